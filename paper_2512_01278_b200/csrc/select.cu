// K3: PillarAttn critical-token selection, one CTA per request.
//   importance[p] = 2^-shift sum_{t < rows} acc[t][p]  (selection.py:207-218, fp64 from the
//                   fixed-point accumulators,
//                   up to the constant 1/(rows*L*Hq) that cannot change order)
//   budget        = max(1, min(ceil(s*n - 1e-9), n))   (selection.py:167-183)
//   positions     = top-budget by value, ties to the lower index, ascending
//                                                     (selection.py:186-204)
// Radix select (8-bit digits, MSB first) finds the budget-th largest key T;
// an ordered block scan then keeps every key > T and the lowest-index keys
// == T until the budget is met, emitting positions already in ascending order.
// Bit-exact with numpy's stable argsort given identical values.
#include <cub/block/block_scan.cuh>

#include "common.cuh"

namespace sd {

constexpr int SEL_THREADS = 1024;

// -0.0 and +0.0 compare equal in numpy's sort, so both map to the +0 key.
__device__ __forceinline__ uint32_t order_key(float v) {
  uint32_t u = __float_as_uint(v == 0.f ? 0.f : v);
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
__device__ __forceinline__ uint64_t order_key(double v) {
  uint64_t u = static_cast<uint64_t>(__double_as_longlong(v == 0.0 ? 0.0 : v));
  return (u & 0x8000000000000000ull) ? ~u : (u | 0x8000000000000000ull);
}

// Same arithmetic as Python: math.ceil(s * n - 1e-9), no FMA contraction.
__device__ __forceinline__ int budget_of(int n, double s) {
  if (n == 0) return 1;
  const double raw = ceil(__dadd_rn(__dmul_rn(s, static_cast<double>(n)), -1e-9));
  long long b = static_cast<long long>(raw);
  if (b > n) b = n;
  return b < 1 ? 1 : static_cast<int>(b);
}

// Select the `take` largest of vals[0..n) into out (ascending positions).
template <typename ValT, typename KeyT>
__device__ void block_topk(const ValT* vals, int n, int take, int32_t* out) {
  using Scan = cub::BlockScan<int, SEL_THREADS>;
  __shared__ typename Scan::TempStorage scan_tmp;
  __shared__ int hist[256];
  __shared__ KeyT s_prefix;
  __shared__ int s_remaining;
  __shared__ int s_carry[2];
  const int tid = threadIdx.x;
  if (take >= n) {
    for (int p = tid; p < n; p += SEL_THREADS) out[p] = p;
    return;
  }
  KeyT prefix = 0, mask = 0;
  int remaining = take;  // rank (1-based) of the threshold among the candidates
  constexpr int BITS = sizeof(KeyT) * 8;
  for (int shift = BITS - 8; shift >= 0; shift -= 8) {
    for (int i = tid; i < 256; i += SEL_THREADS) hist[i] = 0;
    __syncthreads();
    for (int p = tid; p < n; p += SEL_THREADS) {
      const KeyT u = order_key(vals[p]);
      if ((u & mask) == prefix) atomicAdd(&hist[static_cast<int>((u >> shift) & 0xff)], 1);
    }
    __syncthreads();
    if (tid < 32) {
      // warp 0: scan digits from the top; each lane owns 8 consecutive digits
      int local[8];
      int lsum = 0;
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        local[k] = hist[255 - (tid * 8 + k)];
        lsum += local[k];
      }
      int incl = lsum;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int v = __shfl_up_sync(0xffffffffu, incl, o);
        if (tid >= o) incl += v;
      }
      int above = incl - lsum;  // count in higher digits than this lane's block
      const bool here = above < remaining && remaining <= incl;
      if (here) {
        int digit = 255 - tid * 8;
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          if (above + local[k] >= remaining) { digit = 255 - (tid * 8 + k); break; }
          above += local[k];
        }
        s_prefix = prefix | (static_cast<KeyT>(digit) << shift);
        s_remaining = remaining - above;
      }
    }
    __syncthreads();
    prefix = s_prefix;
    remaining = s_remaining;
    mask |= static_cast<KeyT>(0xff) << shift;
    __syncthreads();
  }
  const KeyT T = prefix;
  const int need_eq = remaining;  // elements equal to T to keep, lowest index first
  if (tid == 0) { s_carry[0] = 0; s_carry[1] = 0; }
  __syncthreads();
  for (int base = 0; base < n; base += SEL_THREADS) {
    const int p = base + tid;
    KeyT u = 0;
    if (p < n) u = order_key(vals[p]);
    const int is_eq = (p < n && u == T) ? 1 : 0;
    int eq_before, eq_total;
    Scan(scan_tmp).ExclusiveSum(is_eq, eq_before, eq_total);
    const int eq_rank = s_carry[1] + eq_before;
    const int sel = (p < n && (u > T || (is_eq && eq_rank < need_eq))) ? 1 : 0;
    __syncthreads();
    int sel_before, sel_total;
    Scan(scan_tmp).ExclusiveSum(sel, sel_before, sel_total);
    if (sel) out[s_carry[0] + sel_before] = p;
    __syncthreads();
    if (tid == 0) {
      s_carry[0] += sel_total;
      s_carry[1] += eq_total;
    }
    __syncthreads();
  }
}

__global__ void __launch_bounds__(SEL_THREADS) select_critical_kernel(
    const unsigned long long* __restrict__ acc, int64_t acc_req_stride, int64_t acc_row_stride, double unit,
    const int32_t* __restrict__ n_rows, const int32_t* __restrict__ kv_len, double sparsity,
    const int32_t* __restrict__ req_index, double* __restrict__ imp, int64_t imp_stride, int32_t* __restrict__ crit,
    int64_t crit_stride, int32_t* __restrict__ crit_len, int32_t* __restrict__ budget_out) {
  const int n = kv_len[blockIdx.x];
  const int rows = n_rows[blockIdx.x];
  const int r = req_index ? req_index[blockIdx.x] : blockIdx.x;
  double* v = imp + (int64_t)r * imp_stride;
  const unsigned long long* a = acc + (int64_t)r * acc_req_stride;
  // fixed-point rows -> fp64, summed in row order (deterministic; the reference sums in fp64)
  for (int p = threadIdx.x; p < n; p += SEL_THREADS) {
    double s = 0.0;
    for (int t = 0; t < rows; ++t) s += (double)a[(int64_t)t * acc_row_stride + p] * unit;
    v[p] = s;
  }
  __syncthreads();
  const int b = budget_of(n, sparsity);
  const int take = b < n ? b : n;
  if (threadIdx.x == 0) {
    crit_len[r] = take;
    if (budget_out) budget_out[r] = b;
  }
  block_topk<double, uint64_t>(v, n, take, crit + (int64_t)r * crit_stride);
}

template <typename ValT, typename KeyT>
__global__ void __launch_bounds__(SEL_THREADS) topk_kernel(const ValT* __restrict__ vals, int64_t stride,
                                                           const int32_t* __restrict__ n,
                                                           const int32_t* __restrict__ budget,
                                                           int32_t* __restrict__ out, int64_t out_stride,
                                                           int32_t* __restrict__ out_len) {
  const int r = blockIdx.x;
  const int nn = n[r];
  const int take = budget[r] < nn ? budget[r] : nn;
  if (threadIdx.x == 0) out_len[r] = take;
  block_topk<ValT, KeyT>(vals + (int64_t)r * stride, nn, take, out + (int64_t)r * out_stride);
}

}  // namespace sd

extern "C" int sd_select_critical(const uint64_t* acc, int64_t acc_req_stride, int64_t acc_row_stride,
                                  int32_t acc_shift, const int32_t* n_rows, const int32_t* kv_len, double sparsity,
                                  int32_t num_requests, const int32_t* req_index, double* importance,
                                  int64_t imp_stride, int32_t* crit, int64_t crit_stride, int32_t* crit_len,
                                  int32_t* budget_out, void* stream) {
  SD_REQUIRE(sparsity > 0.0 && sparsity <= 1.0, "sd_select_critical: sparsity must be in (0, 1]");
  SD_REQUIRE(num_requests >= 0, "sd_select_critical: negative request count");
  SD_REQUIRE(acc_shift >= 0 && acc_shift <= 62, "sd_select_critical: acc_shift must be in [0, 62]");
  SD_REQUIRE(acc && n_rows && kv_len && importance && crit && crit_len, "sd_select_critical: null pointer");
  if (num_requests == 0) return 0;
  sd::select_critical_kernel<<<num_requests, sd::SEL_THREADS, 0, static_cast<cudaStream_t>(stream)>>>(
      reinterpret_cast<const unsigned long long*>(acc), acc_req_stride, acc_row_stride, ldexp(1.0, -acc_shift), n_rows,
      kv_len, sparsity, req_index, importance, imp_stride, crit, crit_stride, crit_len, budget_out);
  sd::count_launch();
  SD_CUDA_RETURN();
}

extern "C" int sd_topk(const void* values, int32_t value_dtype, int64_t stride, const int32_t* n,
                       const int32_t* budget, int32_t num, int32_t* out, int64_t out_stride, int32_t* out_len,
                       void* stream) {
  SD_REQUIRE(value_dtype == 0 || value_dtype == 2, "sd_topk: values must be float32 (0) or float64 (2)");
  SD_REQUIRE(values && n && budget && out && out_len, "sd_topk: null pointer");
  if (num <= 0) return 0;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (value_dtype == 0)
    sd::topk_kernel<float, uint32_t><<<num, sd::SEL_THREADS, 0, s>>>(static_cast<const float*>(values), stride, n,
                                                                     budget, out, out_stride, out_len);
  else
    sd::topk_kernel<double, uint64_t><<<num, sd::SEL_THREADS, 0, s>>>(static_cast<const double*>(values), stride,
                                                                      n, budget, out, out_stride, out_len);
  sd::count_launch();
  SD_CUDA_RETURN();
}
