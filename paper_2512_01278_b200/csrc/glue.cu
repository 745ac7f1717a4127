// Glue epilogues around the torch GEMMs (not the attention hot path):
// RMSNorm without gain (model.py:225-226) fused with the cast to the GEMM
// input dtype, so each layer costs one launch per norm instead of five.
#include "common.cuh"

namespace sd {

template <typename T>
__global__ void __launch_bounds__(256) rmsnorm_cast_kernel(const float* __restrict__ x, int h, float eps,
                                                           T* __restrict__ out) {
  const float* xr = x + (int64_t)blockIdx.x * h;
  T* orow = out + (int64_t)blockIdx.x * h;
  float ss = 0.f;
  const bool vec = (h % 4) == 0;
  if (vec) {
    for (int i = threadIdx.x; i < h / 4; i += blockDim.x) {
      const float4 v = reinterpret_cast<const float4*>(xr)[i];
      ss += v.x * v.x + v.y * v.y + v.z * v.z + v.w * v.w;
    }
  } else {
    for (int i = threadIdx.x; i < h; i += blockDim.x) ss += xr[i] * xr[i];
  }
  ss = warp_sum(ss);
  __shared__ float part[8];
  if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = ss;
  __syncthreads();
  if (threadIdx.x < 32) {
    float v = threadIdx.x < (blockDim.x >> 5) ? part[threadIdx.x] : 0.f;
    v = warp_sum(v);
    if (threadIdx.x == 0) part[0] = v;
  }
  __syncthreads();
  const float inv = rsqrtf(part[0] / static_cast<float>(h) + eps);
  for (int i = threadIdx.x; i < h; i += blockDim.x) orow[i] = from_f<T>(xr[i] * inv);
}

}  // namespace sd

extern "C" int sd_rmsnorm_cast(const float* x, int32_t rows, int32_t h, float eps, void* out, int32_t out_dtype,
                               void* stream) {
  SD_REQUIRE(x && out, "sd_rmsnorm_cast: null pointer");
  SD_REQUIRE(rows >= 0 && h >= 1, "sd_rmsnorm_cast: bad shape");
  if (rows == 0) return 0;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (out_dtype == SD_DTYPE_F32)
    sd::rmsnorm_cast_kernel<float><<<rows, 256, 0, s>>>(x, h, eps, static_cast<float*>(out));
  else
    sd::rmsnorm_cast_kernel<__nv_bfloat16><<<rows, 256, 0, s>>>(x, h, eps, static_cast<__nv_bfloat16*>(out));
  sd::count_launch();
  SD_CUDA_RETURN();
}
