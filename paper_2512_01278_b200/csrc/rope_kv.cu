// K5: RoPE epilogue of the QKV projection + paged KV append.
// Restates model.py:212-222 (_rotate: NeoX half split, inv_freq = 1e4^(-2i/d),
// angle at the ABSOLUTE position) and the K/V push of model.py:284-287,
// 326-331, 372-374.  K is stored post-RoPE (drafts gather rotated keys);
// rows go straight into their paged slot (no per-forward buffer copy,
// model.py:271-287's _LayerBuffer is eliminated).
//
// One CTA per row.  cos/sin of the row's angles are computed once in double
// (angle = pos * 10000^(-2i/d), exactly as numpy) into shared memory; the
// (head, pair) rotations are then spread over all threads so consecutive
// threads touch consecutive elements.  fp32 parity mode rotates in double.
#include "common.cuh"

#include <algorithm>

namespace sd {

template <typename T>
__global__ void __launch_bounds__(256) rope_kv_kernel(const T* __restrict__ qkv, int64_t row_stride,
                                                      const int32_t* __restrict__ row_table,
                                                      const int32_t* __restrict__ row_pos, PagedKv kv,
                                                      int layer, int q_heads, T* __restrict__ q_out) {
  extern __shared__ double cs[];  // [half] cos, [half] sin
  const int r = blockIdx.x;
  const int D = kv.head_dim, half = D / 2, Hkv = kv.kv_heads;
  const int pos = row_pos[r];
  const int64_t slot = kv.slot_of(row_table[r], pos);
  const T* x = qkv + (int64_t)r * row_stride;
  T* K = static_cast<T*>(const_cast<void*>(kv.k)) + (int64_t)layer * kv.layer_stride;
  T* V = static_cast<T*>(const_cast<void*>(kv.v)) + (int64_t)layer * kv.layer_stride;
  for (int i = threadIdx.x; i < half; i += blockDim.x) {
    const double inv = pow(10000.0, -static_cast<double>(2 * i) / static_cast<double>(D));
    double s, c;
    sincos(static_cast<double>(pos) * inv, &s, &c);
    cs[i] = c;
    cs[half + i] = s;
  }
  __syncthreads();
  const int pairs = (q_heads + Hkv) * half;
  for (int idx = threadIdx.x; idx < pairs; idx += blockDim.x) {
    const int hq = idx / half, i = idx - hq * half;
    const T* src = x + hq * D;
    float lo, hi;
    if constexpr (sizeof(T) == 4) {  // parity mode: rotate in double, round once
      const double a = to_f(src[i]), b = to_f(src[i + half]);
      lo = static_cast<float>(a * cs[i] - b * cs[half + i]);
      hi = static_cast<float>(a * cs[half + i] + b * cs[i]);
    } else {
      const float a = to_f(src[i]), b = to_f(src[i + half]);
      const float cf = static_cast<float>(cs[i]), sf = static_cast<float>(cs[half + i]);
      lo = a * cf - b * sf;
      hi = a * sf + b * cf;
    }
    T* dst = hq < q_heads ? q_out + ((int64_t)r * q_heads + hq) * D : K + kv.row_off(slot, hq - q_heads);
    dst[i] = from_f<T>(lo);
    dst[i + half] = from_f<T>(hi);
  }
  const T* vsrc = x + (q_heads + Hkv) * D;
  T* vdst = V + kv.row_off(slot, 0);
  const int n = Hkv * D;
  if ((n * sizeof(T)) % 16 == 0 && (reinterpret_cast<uintptr_t>(vsrc) % 16) == 0) {
    const int nv = n * sizeof(T) / 16;
    for (int j = threadIdx.x; j < nv; j += blockDim.x)
      reinterpret_cast<uint4*>(vdst)[j] = reinterpret_cast<const uint4*>(vsrc)[j];
  } else {
    for (int j = threadIdx.x; j < n; j += blockDim.x) vdst[j] = vsrc[j];
  }
}

// cos/sin of every row's angles, once per forward (all layers share the positions):
// table[r][i] = (cos, sin)(pos_r * 10000^(-2i/d)), computed in double like the per-layer path
__global__ void rope_table_kernel(const int32_t* __restrict__ row_pos, int rows, int half, int D,
                                  float2* __restrict__ table) {
  const int64_t n = (int64_t)rows * half;
  for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < n; idx += (int64_t)gridDim.x * blockDim.x) {
    const int r = static_cast<int>(idx / half), i = static_cast<int>(idx - (int64_t)r * half);
    const double inv = pow(10000.0, -static_cast<double>(2 * i) / static_cast<double>(D));
    double sn, cs;
    sincos(static_cast<double>(row_pos[r]) * inv, &sn, &cs);
    table[idx] = make_float2(static_cast<float>(cs), static_cast<float>(sn));
  }
}

// bf16 K5 with the precomputed table: 8 bf16 pairs (16 B of each half) per thread, rows
// spread over the grid so every thread has work
// one CTA per row, one thread per 8-element group of a head half: the q / k groups are
// rotated with the row's cos/sin (two 16-byte table loads per 4 pairs), the v row is copied;
// the block-table lookup (only the k and v stores need it) overlaps the loads
__global__ void __launch_bounds__(320) rope_kv_table_kernel(const __nv_bfloat16* __restrict__ qkv, int64_t row_stride,
                                                            const int32_t* __restrict__ row_table,
                                                            const int32_t* __restrict__ row_pos, PagedKv kv, int layer,
                                                            int q_heads, const float2* __restrict__ table,
                                                            __nv_bfloat16* __restrict__ q_out) {
  const int r = blockIdx.x;
  const int D = kv.head_dim, half = D / 2, Hkv = kv.kv_heads;
  const __nv_bfloat16* x = qkv + (int64_t)r * row_stride;
  const int vec_per_head = half / 8;                    // 8-element groups per half
  const int groups = (q_heads + Hkv) * vec_per_head;
  const int vgroups = Hkv * D / 8;                      // 16-byte pieces of the v row
  const int table_row = row_table[r];
  const int pos = row_pos[r];
  const int64_t slot = (kv.slot_of(table_row, pos));
  __nv_bfloat16* K = static_cast<__nv_bfloat16*>(const_cast<void*>(kv.k)) + (int64_t)layer * kv.layer_stride;
  __nv_bfloat16* V = static_cast<__nv_bfloat16*>(const_cast<void*>(kv.v)) + (int64_t)layer * kv.layer_stride;
  const float4* tr = reinterpret_cast<const float4*>(table + (int64_t)r * half);
  for (int gi = threadIdx.x; gi < groups + vgroups; gi += blockDim.x) {
    if (gi >= groups) {  // v: plain copy into the paged slot
      const int j = gi - groups;
      reinterpret_cast<uint4*>(V + kv.row_off(slot, 0))[j] = reinterpret_cast<const uint4*>(x + (q_heads + Hkv) * D)[j];
      continue;
    }
    const int hq = gi / vec_per_head, i0 = (gi - hq * vec_per_head) * 8;
    const __nv_bfloat16* src = x + hq * D;
    const uint4 lo_raw = *reinterpret_cast<const uint4*>(src + i0);
    const uint4 hi_raw = *reinterpret_cast<const uint4*>(src + half + i0);
    float4 cs4[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) cs4[j] = __ldg(tr + i0 / 2 + j);  // (cos, sin) of pairs i0 .. i0 + 7
    const float2* cs = reinterpret_cast<const float2*>(cs4);
    const __nv_bfloat16* lo = reinterpret_cast<const __nv_bfloat16*>(&lo_raw);
    const __nv_bfloat16* hi = reinterpret_cast<const __nv_bfloat16*>(&hi_raw);
    uint4 olo_raw, ohi_raw;
    __nv_bfloat16* olo = reinterpret_cast<__nv_bfloat16*>(&olo_raw);
    __nv_bfloat16* ohi = reinterpret_cast<__nv_bfloat16*>(&ohi_raw);
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const float a = __bfloat162float(lo[j]), b = __bfloat162float(hi[j]);
      olo[j] = __float2bfloat16_rn(a * cs[j].x - b * cs[j].y);
      ohi[j] = __float2bfloat16_rn(a * cs[j].y + b * cs[j].x);
    }
    __nv_bfloat16* dst = hq < q_heads ? q_out + ((int64_t)r * q_heads + hq) * D : K + kv.row_off(slot, hq - q_heads);
    *reinterpret_cast<uint4*>(dst + i0) = olo_raw;
    *reinterpret_cast<uint4*>(dst + half + i0) = ohi_raw;
  }
}

int rope_table(const int32_t* row_pos, int rows, int head_dim, float2* table, cudaStream_t s) {
  const int half = head_dim / 2;
  const int64_t n = (int64_t)rows * half;
  const int blocks = (int)std::min<int64_t>((n + 255) / 256, 148 * 4);
  rope_table_kernel<<<blocks, 256, 0, s>>>(row_pos, rows, half, head_dim, table);
  count_launch();
  return 0;
}

// bf16 K5 through a rope_table; head_dim must be a multiple of 16 and rows 16-byte aligned
int rope_kv_write_table(const void* qkv, int64_t qkv_row_stride, int rows, const int32_t* row_table,
                        const int32_t* row_pos, const sd_paged_kv* kv, int layer, int q_heads, const float2* table,
                        void* q_out, cudaStream_t s) {
  PagedKv p = make_paged(kv);
  rope_kv_table_kernel<<<rows, 320, 0, s>>>(static_cast<const __nv_bfloat16*>(qkv), qkv_row_stride, row_table,
                                            row_pos, p, layer, q_heads, table, static_cast<__nv_bfloat16*>(q_out));
  count_launch();
  return 0;
}

}  // namespace sd

extern "C" int sd_rope_kv_write(const void* qkv, int64_t qkv_row_stride, int32_t rows,
                                const int32_t* row_table, const int32_t* row_pos, const sd_paged_kv* kv,
                                int32_t layer, int32_t q_heads, void* q_out, void* stream) {
  SD_REQUIRE(kv != nullptr && qkv != nullptr && q_out != nullptr, "sd_rope_kv_write: null pointer");
  SD_REQUIRE(rows >= 0, "sd_rope_kv_write: negative row count");
  SD_REQUIRE(kv->head_dim % 2 == 0, "sd_rope_kv_write: head_dim must be even");
  SD_REQUIRE(q_heads % kv->kv_heads == 0, "sd_rope_kv_write: kv_heads must divide q_heads");
  if (rows == 0) return 0;
  sd::PagedKv p = sd::make_paged(kv);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const size_t smem = sizeof(double) * kv->head_dim;
  if (kv->dtype == SD_DTYPE_F32)
    sd::rope_kv_kernel<float><<<rows, 256, smem, s>>>(static_cast<const float*>(qkv), qkv_row_stride, row_table,
                                                     row_pos, p, layer, q_heads, static_cast<float*>(q_out));
  else
    sd::rope_kv_kernel<__nv_bfloat16><<<rows, 256, smem, s>>>(static_cast<const __nv_bfloat16*>(qkv),
                                                             qkv_row_stride, row_table, row_pos, p, layer,
                                                             q_heads, static_cast<__nv_bfloat16*>(q_out));
  sd::count_launch();
  SD_CUDA_RETURN();
}
