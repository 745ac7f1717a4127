// K4: greedy targets and the verification accept rule.
//   argmax with ties to the lowest token id           (model.py:388-390)
//   accepted = longest prefix with drafted[i] == target[i];
//   bonus = target[accepted]                           (engine.py:231-239)
#include "common.cuh"

namespace sd {

constexpr int AM_THREADS = 256;

template <typename A>
__device__ __forceinline__ void better(A& bv, int& bi, A v, int i) {
  if (v > bv || (v == bv && i < bi)) {
    bv = v;
    bi = i;
  }
}

__device__ __forceinline__ double to_acc(double x) { return x; }
__device__ __forceinline__ float to_acc(float x) { return x; }
__device__ __forceinline__ float to_acc(__nv_bfloat16 x) { return __bfloat162float(x); }

// T = logits dtype, A = comparison type (fp64 rows compare in fp64: no tie created by rounding)
template <typename T, typename A>
__global__ void __launch_bounds__(AM_THREADS) argmax_kernel(const T* __restrict__ logits, int64_t stride,
                                                            int vocab, int32_t* __restrict__ out) {
  const T* row = logits + (int64_t)blockIdx.x * stride;
  A bv = -INFINITY;
  int bi = 0x7fffffff;
  constexpr int VEC = 16 / sizeof(T);
  const bool aligned = (reinterpret_cast<uintptr_t>(row) % 16) == 0;
  int start = 0;
  if (aligned) {
    const int nvec = vocab / VEC;
    for (int i = threadIdx.x; i < nvec; i += AM_THREADS) {
      const uint4 raw = reinterpret_cast<const uint4*>(row)[i];
      const T* e = reinterpret_cast<const T*>(&raw);
#pragma unroll
      for (int k = 0; k < VEC; ++k) better(bv, bi, to_acc(e[k]), i * VEC + k);
    }
    start = nvec * VEC;
  }
  for (int i = start + threadIdx.x; i < vocab; i += AM_THREADS) better(bv, bi, to_acc(row[i]), i);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const A ov = __shfl_xor_sync(0xffffffffu, bv, o);
    const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
    better(bv, bi, ov, oi);
  }
  __shared__ A sv[AM_THREADS / 32];
  __shared__ int si[AM_THREADS / 32];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) {
    sv[warp] = bv;
    si[warp] = bi;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < AM_THREADS / 32; ++w) better(bv, bi, sv[w], si[w]);
    out[blockIdx.x] = bi == 0x7fffffff ? 0 : bi;
  }
}

__global__ void accept_kernel(const int32_t* __restrict__ targets, const int32_t* __restrict__ tokens,
                              const int32_t* __restrict__ row0, const int32_t* __restrict__ nrows, int num,
                              int32_t* __restrict__ accepted, int32_t* __restrict__ bonus) {
  const int m = blockIdx.x * blockDim.x + threadIdx.x;
  if (m >= num) return;
  const int r0 = row0[m], n = nrows[m];
  int a = 0;
  while (a < n - 1 && tokens[r0 + 1 + a] == targets[r0 + a]) ++a;
  accepted[m] = a;
  bonus[m] = targets[r0 + a];
}

}  // namespace sd

extern "C" int sd_argmax_rows(const void* logits, int32_t dtype, int64_t row_stride, int32_t rows, int32_t vocab,
                              int32_t* out, void* stream) {
  SD_REQUIRE(logits && out, "sd_argmax_rows: null pointer");
  SD_REQUIRE(vocab >= 1 && rows >= 0, "sd_argmax_rows: bad shape");
  if (rows == 0) return 0;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  SD_REQUIRE(dtype == SD_DTYPE_F32 || dtype == SD_DTYPE_BF16 || dtype == SD_DTYPE_F64,
             "sd_argmax_rows: logits must be float32, bfloat16 or float64");
  if (dtype == SD_DTYPE_F32)
    sd::argmax_kernel<float, float><<<rows, sd::AM_THREADS, 0, s>>>(static_cast<const float*>(logits), row_stride,
                                                                    vocab, out);
  else if (dtype == SD_DTYPE_F64)
    sd::argmax_kernel<double, double><<<rows, sd::AM_THREADS, 0, s>>>(static_cast<const double*>(logits), row_stride,
                                                                      vocab, out);
  else
    sd::argmax_kernel<__nv_bfloat16, float><<<rows, sd::AM_THREADS, 0, s>>>(
        static_cast<const __nv_bfloat16*>(logits), row_stride, vocab, out);
  sd::count_launch();
  SD_CUDA_RETURN();
}

extern "C" int sd_greedy_accept(const int32_t* targets, const int32_t* tokens, const int32_t* row0,
                                const int32_t* nrows, int32_t num, int32_t* accepted, int32_t* bonus, void* stream) {
  SD_REQUIRE(targets && tokens && row0 && nrows && accepted && bonus, "sd_greedy_accept: null pointer");
  if (num <= 0) return 0;
  sd::accept_kernel<<<(num + 127) / 128, 128, 0, static_cast<cudaStream_t>(stream)>>>(targets, tokens, row0, nrows,
                                                                                      num, accepted, bonus);
  sd::count_launch();
  SD_CUDA_RETURN();
}
