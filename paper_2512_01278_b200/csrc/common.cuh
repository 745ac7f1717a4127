// Shared device/host helpers for the spardec B200 kernels (sm_100a only).
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdio>
#include <string>

#include "../../include/spardec_b200.h"

namespace sd {

// ---- error plumbing (host) ---------------------------------------------------
void set_error(const std::string& msg);
void count_launch(int n = 1);

#define SD_REQUIRE(cond, msg)      \
  do {                             \
    if (!(cond)) {                 \
      ::sd::set_error(msg);        \
      return -1;                   \
    }                              \
  } while (0)

#define SD_CUDA_RETURN()                                               \
  do {                                                                 \
    cudaError_t _e = cudaGetLastError();                               \
    if (_e != cudaSuccess) {                                           \
      ::sd::set_error(std::string("CUDA: ") + cudaGetErrorString(_e)); \
      return (int)_e;                                                  \
    }                                                                  \
    return 0;                                                          \
  } while (0)

// ---- K5 helpers shared by forward.cu (rope_kv.cu) ------------------------------------
inline int64_t rope_table_bytes(int rows, int head_dim) { return ((int64_t)rows * (head_dim / 2) * 8 + 255) / 256 * 256; }
int rope_table(const int32_t* row_pos, int rows, int head_dim, float2* table, cudaStream_t s);
int rope_kv_write_table(const void* qkv, int64_t qkv_row_stride, int rows, const int32_t* row_table,
                        const int32_t* row_pos, const sd_paged_kv* kv, int layer, int q_heads, const float2* table,
                        void* q_out, cudaStream_t s);

// ---- element conversions ------------------------------------------------------
template <typename T>
__device__ __forceinline__ float to_f(T x);
template <>
__device__ __forceinline__ float to_f<float>(float x) { return x; }
template <>
__device__ __forceinline__ float to_f<__nv_bfloat16>(__nv_bfloat16 x) { return __bfloat162float(x); }

template <typename T>
__device__ __forceinline__ T from_f(float x);
template <>
__device__ __forceinline__ float from_f<float>(float x) { return x; }
template <>
__device__ __forceinline__ __nv_bfloat16 from_f<__nv_bfloat16>(float x) { return __float2bfloat16_rn(x); }

// ---- paged KV addressing ---------------------------------------------------------
// Page = 2^page_shift tokens; logical position -> physical slot through the
// request's block-table row (kvpool.py:1-8: one logical page per token, grouped
// into physical pages so dense verify reads stream contiguously).
struct PagedKv {
  const void* k;
  const void* v;
  int64_t layer_stride;
  const int32_t* table;
  int32_t table_stride;
  int32_t page_shift;
  int32_t kv_heads;
  int32_t head_dim;

  __device__ __forceinline__ int64_t slot_of(int32_t table_row, int32_t pos) const {
    const int32_t page = __ldg(table + (int64_t)table_row * table_stride + (pos >> page_shift));
    return ((int64_t)page << page_shift) | (pos & ((1 << page_shift) - 1));
  }
  // element offset of (slot, head) within one layer
  __device__ __forceinline__ int64_t row_off(int64_t slot, int32_t head) const {
    return (slot * kv_heads + head) * (int64_t)head_dim;
  }
};

inline PagedKv make_paged(const sd_paged_kv* p) {
  PagedKv r;
  r.k = p->k;
  r.v = p->v;
  r.layer_stride = p->layer_stride;
  r.table = p->block_table;
  r.table_stride = p->table_stride;
  r.page_shift = p->page_shift;
  r.kv_heads = p->kv_heads;
  r.head_dim = p->head_dim;
  return r;
}

// ---- attention work item -----------------------------------------------------------
struct Item {
  int table_row, q_row0, nq, qpos0, crit_off, crit_len, dense_lo, acc_row, acc_step;
  __device__ __forceinline__ int num_keys() const { return crit_len + (qpos0 + nq - dense_lo); }
  // absolute position of key j (critical list first, then the dense range)
  __device__ __forceinline__ int key_pos(const int32_t* crit, int j) const {
    return j < crit_len ? __ldg(crit + crit_off + j) : dense_lo + (j - crit_len);
  }
};

__device__ __forceinline__ Item load_item(const int32_t* items, int i) {
  const int32_t* p = items + (int64_t)i * SD_ITEM_FIELDS;
  Item it;
  it.table_row = p[SD_ITEM_TABLE_ROW];
  it.q_row0 = p[SD_ITEM_Q_ROW0];
  it.nq = p[SD_ITEM_NQ];
  it.qpos0 = p[SD_ITEM_QPOS0];
  it.crit_off = p[SD_ITEM_CRIT_OFF];
  it.crit_len = p[SD_ITEM_CRIT_LEN];
  it.dense_lo = p[SD_ITEM_DENSE_LO];
  it.acc_row = p[SD_ITEM_ACC_ROW];
  it.acc_step = p[SD_ITEM_ACC_STEP];
  return it;
}

// planted-concentration bonus (model.py:246-247,256-262): sorted list, binary search
__device__ __forceinline__ float planted_bias(const int32_t* planted, int n, float bonus, int pos) {
  if (n == 0) return 0.f;
  int lo = 0, hi = n;
  while (lo < hi) {
    int mid = (lo + hi) >> 1;
    int v = __ldg(planted + mid);
    if (v < pos) lo = mid + 1; else hi = mid;
  }
  return (lo < n && __ldg(planted + lo) == pos) ? bonus : 0.f;
}

__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

}  // namespace sd
