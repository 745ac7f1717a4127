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

// the row stays in registers (h <= 256 * 4 * NV, h % 1024 == 0): one read of x, one write
template <int NV>
__global__ void __launch_bounds__(256) rmsnorm_cast_reg_kernel(const float* __restrict__ x, int h, float eps,
                                                               __nv_bfloat16* __restrict__ out) {
  const float4* xr = reinterpret_cast<const float4*>(x + (int64_t)blockIdx.x * h);
  float4 v[NV];
  const int n4 = h / 4;
  float ss = 0.f;
#pragma unroll
  for (int j = 0; j < NV; ++j) {
    const int i = j * 256 + threadIdx.x;
    v[j] = i < n4 ? xr[i] : make_float4(0.f, 0.f, 0.f, 0.f);
    ss += v[j].x * v[j].x + v[j].y * v[j].y + v[j].z * v[j].z + v[j].w * v[j].w;
  }
  ss = warp_sum(ss);
  __shared__ float part[8];
  if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = ss;
  __syncthreads();
  float tot = 0.f;
#pragma unroll
  for (int w = 0; w < 8; ++w) tot += part[w];
  const float inv = rsqrtf(tot / static_cast<float>(h) + eps);
  uint2* orow = reinterpret_cast<uint2*>(out + (int64_t)blockIdx.x * h);
#pragma unroll
  for (int j = 0; j < NV; ++j) {
    const int i = j * 256 + threadIdx.x;
    if (i < n4) {
      __nv_bfloat162 a = __floats2bfloat162_rn(v[j].x * inv, v[j].y * inv);
      __nv_bfloat162 b = __floats2bfloat162_rn(v[j].z * inv, v[j].w * inv);
      orow[i] = make_uint2(*reinterpret_cast<uint32_t*>(&a), *reinterpret_cast<uint32_t*>(&b));
    }
  }
}

}  // namespace sd

extern "C" int sd_rmsnorm_cast(const float* x, int32_t rows, int32_t h, float eps, void* out, int32_t out_dtype,
                               void* stream) {
  SD_REQUIRE(x && out, "sd_rmsnorm_cast: null pointer");
  SD_REQUIRE(rows >= 0 && h >= 1, "sd_rmsnorm_cast: bad shape");
  if (rows == 0) return 0;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const bool aligned = (reinterpret_cast<uintptr_t>(x) % 16) == 0 && (reinterpret_cast<uintptr_t>(out) % 8) == 0;
  if (out_dtype == SD_DTYPE_BF16 && aligned && h % 1024 == 0 && h <= 8192) {
    auto* o = static_cast<__nv_bfloat16*>(out);
    if (h <= 4096)
      sd::rmsnorm_cast_reg_kernel<4><<<rows, 256, 0, s>>>(x, h, eps, o);
    else
      sd::rmsnorm_cast_reg_kernel<8><<<rows, 256, 0, s>>>(x, h, eps, o);
  } else if (out_dtype == SD_DTYPE_F32)
    sd::rmsnorm_cast_kernel<float><<<rows, 256, 0, s>>>(x, h, eps, static_cast<float*>(out));
  else
    sd::rmsnorm_cast_kernel<__nv_bfloat16><<<rows, 256, 0, s>>>(x, h, eps, static_cast<__nv_bfloat16*>(out));
  sd::count_launch();
  SD_CUDA_RETURN();
}
