// Generic (FFMA) grouped-query attention with exact two-phase softmax and
// PillarAttn score emission.  Used for fp32 parity mode and head dims the
// tensor-core kernel does not cover.  Restates model.py:229-253 (_attend) for
// every query row of a work item: logits = q.k / sqrt(d) (+ planted bonus),
// max-subtracted softmax, ctx = P.V, lse = log(sum) + max; scores
// acc[row][pos] += sum_{h in group} exp(logit - lse)  (selection.py:78-135).
#include "common.cuh"

namespace sd {

template <typename T>
__global__ void __launch_bounds__(256) attn_generic_kernel(
    const T* __restrict__ q, T* __restrict__ out, float* __restrict__ lse_out, PagedKv kv,
    int layer, const int32_t* __restrict__ items, const int32_t* __restrict__ crit,
    unsigned long long* __restrict__ acc, int64_t acc_stride, float acc_scale, const int32_t* __restrict__ planted,
    int n_planted, float bonus, int q_heads, float inv_sqrt_d, float* __restrict__ ws,
    int max_keys, int max_rows) {
  const Item it = load_item(items, blockIdx.y);
  const int h = blockIdx.x;
  const int G = q_heads / kv.kv_heads;
  const int D = kv.head_dim;
  const int R = it.nq * G;
  const int Nk = it.num_keys();
  const int tid = threadIdx.x, nthr = blockDim.x;
  const int lane = tid & 31, warp = tid >> 5, nwarp = nthr >> 5;

  float* S = ws + ((int64_t)blockIdx.y * kv.kv_heads + h) * ((int64_t)max_rows * max_keys + 3 * max_keys);
  int32_t* kpos = reinterpret_cast<int32_t*>(S + (int64_t)max_rows * max_keys);
  int32_t* kslot = kpos + max_keys;
  float* kbias = reinterpret_cast<float*>(kslot + max_keys);

  // Logits are kept WITHOUT the planted bonus and the bonus is carried
  // separately, so exponents (s - s_max) + (b - b_max) stay exact in fp32
  // even with the +2000 bonus (the reference computes in fp64).
  extern __shared__ float smem[];
  float* sq = smem;            // [R][D]
  float* sms = sq + R * D;     // [R] logit of the row max
  float* smb = sms + R;        // [R] bonus of the row max
  float* sll = smb + R;        // [R] log(sum)

  const T* K = static_cast<const T*>(kv.k) + (int64_t)layer * kv.layer_stride;
  const T* V = static_cast<const T*>(kv.v) + (int64_t)layer * kv.layer_stride;

  for (int i = tid; i < R * D; i += nthr) {
    const int r = i / D, d = i - r * D;
    const int qt = r / G, g = r - qt * G;
    sq[i] = to_f(q[((int64_t)(it.q_row0 + qt) * q_heads + h * G + g) * D + d]);
  }
  for (int j = tid; j < Nk; j += nthr) {
    const int pos = it.key_pos(crit, j);
    kpos[j] = pos;
    kslot[j] = (int32_t)kv.slot_of(it.table_row, pos);
    kbias[j] = planted_bias(planted, n_planted, bonus, pos);
  }
  __syncthreads();

  // phase 1: every visible logit of every row
  for (int i = tid; i < R * Nk; i += nthr) {
    const int r = i / Nk, j = i - r * Nk;
    const int pos = kpos[j];
    const bool vis = (j < it.crit_len) || (pos <= it.qpos0 + r / G);
    float s = -INFINITY;
    if (vis) {
      const T* kr = K + kv.row_off(kslot[j], h);
      const float* qr = sq + r * D;
      float dot = 0.f;
      for (int d = 0; d < D; ++d) dot = fmaf(qr[d], to_f(kr[d]), dot);
      s = dot * inv_sqrt_d;
    }
    S[(int64_t)r * max_keys + j] = s;
  }
  __syncthreads();

  // per-row log-sum-exp around the (logit, bonus) pair of the row max
  for (int r = warp; r < R; r += nwarp) {
    const float* Sr = S + (int64_t)r * max_keys;
    float m = -INFINITY;
    int arg = 0x7fffffff;
    for (int j = lane; j < Nk; j += 32) {
      const float t = Sr[j] + kbias[j];
      if (t > m) { m = t; arg = j; }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const float om = __shfl_xor_sync(0xffffffffu, m, o);
      const int oa = __shfl_xor_sync(0xffffffffu, arg, o);
      if (om > m || (om == m && oa < arg)) { m = om; arg = oa; }
    }
    const float ms = Sr[arg], mb = kbias[arg];
    float l = 0.f;
    for (int j = lane; j < Nk; j += 32) l += expf((Sr[j] - ms) + (kbias[j] - mb));
    l = warp_sum(l);
    const float ll = logf(l);
    if (lane == 0) {
      sms[r] = ms;
      smb[r] = mb;
      sll[r] = ll;
      if (lse_out) lse_out[(int64_t)(it.q_row0 + r / G) * q_heads + h * G + r % G] = (ms + mb) + ll;
    }
  }
  __syncthreads();

  // phase 2: ctx = P.V
  for (int i = tid; i < R * D; i += nthr) {
    const int r = i / D, d = i - r * D;
    const float* Sr = S + (int64_t)r * max_keys;
    const float ms = sms[r], mb = smb[r], ll = sll[r];
    float o = 0.f;
    for (int j = 0; j < Nk; ++j) {
      const float s = Sr[j];
      if (s == -INFINITY) continue;
      o = fmaf(expf(((s - ms) + (kbias[j] - mb)) - ll), to_f(V[kv.row_off(kslot[j], h) + d]), o);
    }
    const int qt = r / G, g = r - qt * G;
    out[((int64_t)(it.q_row0 + qt) * q_heads + h * G + g) * D + d] = from_f<T>(o);
  }

  // score emission: one atomic per (query token, key) summed over the group
  if (acc != nullptr && it.acc_row >= 0) {
    for (int i = tid; i < it.nq * Nk; i += nthr) {
      const int qt = i / Nk, j = i - qt * Nk;
      float sum = 0.f;
      for (int g = 0; g < G; ++g) {
        const int r = qt * G + g;
        const float s = S[(int64_t)r * max_keys + j];
        if (s != -INFINITY) sum += expf(((s - sms[r]) + (kbias[j] - smb[r])) - sll[r]);
      }
      // fixed point (spardec_b200.h): order-independent integer accumulation
      const unsigned long long u = __float2ull_rn(sum * acc_scale);
      if (u != 0ull) atomicAdd(acc + (int64_t)(it.acc_row + qt * it.acc_step) * acc_stride + kpos[j], u);
    }
  }
}

int64_t generic_ws_bytes(int num_items, int max_keys, int max_rows, int kv_heads) {
  return (int64_t)num_items * kv_heads * ((int64_t)max_rows * max_keys + 3 * max_keys) * 4;
}

int launch_attn_generic(const void* q, void* out, float* lse, const sd_paged_kv* kvp, int layer,
                        const int32_t* items, int num_items, int max_keys, int max_nq,
                        const int32_t* crit, unsigned long long* acc, int64_t acc_stride, int acc_shift,
                        const int32_t* planted,
                        int n_planted, float bonus, int q_heads, float scale, void* ws,
                        int64_t ws_bytes, cudaStream_t stream) {
  const int G = q_heads / kvp->kv_heads;
  const int max_rows = max_nq * G;
  SD_REQUIRE(ws_bytes >= generic_ws_bytes(num_items, max_keys, max_rows, kvp->kv_heads),
             "sd_attention: workspace too small for the generic kernel");
  const size_t smem = ((size_t)max_rows * kvp->head_dim + 3 * max_rows) * sizeof(float);
  SD_REQUIRE(smem <= 200 * 1024, "sd_attention: generic kernel query tile exceeds shared memory");
  PagedKv kv = make_paged(kvp);
  dim3 grid(kvp->kv_heads, num_items);
  if (kvp->dtype == SD_DTYPE_F32) {
    if (smem > 48 * 1024)
      cudaFuncSetAttribute(attn_generic_kernel<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attn_generic_kernel<float><<<grid, 256, smem, stream>>>(
        static_cast<const float*>(q), static_cast<float*>(out), lse, kv, layer, items, crit, acc,
        acc_stride, ldexpf(1.f, acc_shift), planted, n_planted, bonus, q_heads, scale, static_cast<float*>(ws), max_keys, max_rows);
  } else {
    if (smem > 48 * 1024)
      cudaFuncSetAttribute(attn_generic_kernel<__nv_bfloat16>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attn_generic_kernel<__nv_bfloat16><<<grid, 256, smem, stream>>>(
        static_cast<const __nv_bfloat16*>(q), static_cast<__nv_bfloat16*>(out), lse, kv, layer, items,
        crit, acc, acc_stride, ldexpf(1.f, acc_shift), planted, n_planted, bonus, q_heads, scale, static_cast<float*>(ws),
        max_keys, max_rows);
  }
  count_launch();
  // workspace contract (spardec_b200.h): handed back zero-filled
  cudaMemsetAsync(ws, 0, generic_ws_bytes(num_items, max_keys, max_rows, kvp->kv_heads), stream);
  SD_CUDA_RETURN();
}

}  // namespace sd
