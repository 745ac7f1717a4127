// Tensor-core (bf16 mma.sync m16n8k16) paged attention for sm_100a with a
// thread-block cluster per (work item, kv head) and an exact two-pass softmax.
//
//   grid    = (C, kv_heads, num_items), cluster = (C, 1, 1)
//   CTA c   = keys [c*chunk, (c+1)*chunk) of the item's key list
//             (critical positions first, then the dense causal range)
//
// setup    the chunk's key positions and physical slots are resolved ONCE into
//          shared memory (block table + critical list), so every later
//          16-byte cp.async is one smem broadcast read + one address FMA.
// pass 1   K tiles (64 keys x d) stream HBM -> smem through a cp.async ring
//          (L2 evict_last); S = Q K^T on tensor cores (rows = query token x
//          GQA group); every thread keeps an online (max, sum) for its rows.
// exchange (max, sum) across the cluster through DSMEM -> exact row lse.
// pass 2   K (L2-resident re-read) + V tiles; each warp recomputes S for 16
//          keys, P = exp2(S - lse) is FINAL and stays in registers: its
//          m16n8 accumulator fragments ARE the m16k16 A fragments of P V, so
//          no shared-memory round trip and no extra barrier.  PillarAttn's
//          score accumulator acc[token][pos] += sum_{g in group} P is emitted
//          from the same registers (warp shuffles over the group's rows).
// reduce   per-warp O partials -> smem -> summed across the cluster through
//          DSMEM, written once.
//
// HBM traffic = K + V once per (item, kv head); logits never leave the SM
// (SURVEY.md §7.2 option (c)); two CTAs per SM; any context length.
//
// Restates model.py:229-253 (_attend), used by forward_full (verify, prefill;
// model.py:318-334) and forward_sparse (draft; model.py:360-380), and the
// score path selection.py:78-135.
#include <cooperative_groups.h>

#include "common.cuh"

namespace cg = cooperative_groups;

namespace sd {
namespace mma_attn {

constexpr int TK = 64;   // keys per tile
constexpr int NT = 256;  // threads per CTA
constexpr int NW = NT / 32;
constexpr float LOG2E = 1.4426950408889634f;
constexpr float LN2 = 0.6931471805599453f;

__device__ __forceinline__ uint64_t policy_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;\n" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;\n" : "=l"(p));
  return p;
}
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, int src_bytes, uint64_t policy) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.cg.shared.global.L2::cache_hint [%0], [%1], 16, %2, %3;\n" ::"r"(s), "l"(gmem),
               "r"(src_bytes), "l"(policy));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

__device__ __forceinline__ void ldsm_x4(unsigned& r0, unsigned& r1, unsigned& r2, unsigned& r3, const void* p) {
  const unsigned a = static_cast<unsigned>(__cvta_generic_to_shared(p));
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];\n"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3) : "r"(a));
}
__device__ __forceinline__ void ldsm_x4_t(unsigned& r0, unsigned& r1, unsigned& r2, unsigned& r3, const void* p) {
  const unsigned a = static_cast<unsigned>(__cvta_generic_to_shared(p));
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];\n"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3) : "r"(a));
}
__device__ __forceinline__ void mma_bf16(float (&c)[4], unsigned a0, unsigned a1, unsigned a2, unsigned a3,
                                         unsigned b0, unsigned b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};\n"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}
__device__ __forceinline__ unsigned pack_bf16(float lo, float hi) {
  __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<unsigned*>(&v);
}

struct Params {
  const __nv_bfloat16* q;
  __nv_bfloat16* out;
  float* lse_out;
  PagedKv kv;
  int layer;
  const int32_t* items;
  const int32_t* crit;
  float* acc;
  int64_t acc_stride;
  const int32_t* planted;
  int n_planted;
  float bonus_log2;
  int q_heads;
  float scale_log2;
  int chunk;  // keys per CTA, multiple of TK
};

// Shared-memory carve, identical on host and device.
struct Layout {
  int ring_off, q_off, pos_off, slot_off, wm_off, wl_off, m_off, l_off, lse_off, total;
};
__host__ __device__ inline Layout make_layout(int D, int MT, int nslot, int chunk) {
  const int RP = MT * 16;
  const int krow = D + 8;
  Layout L;
  int o = 0;
  L.ring_off = o;
  {
    const int ring = nslot * TK * krow * 2;
    const int obuf = RP * D * 4;  // O partials reuse the ring after the loop
    o += ring > obuf ? ring : obuf;
  }
  L.q_off = o;    o += RP * krow * 2;
  L.pos_off = o;  o += chunk * 4;
  L.slot_off = o; o += chunk * 4;
  L.wm_off = o;   o += NW * RP * 4;
  L.wl_off = o;   o += NW * RP * 4;
  L.m_off = o;    o += RP * 4;
  L.l_off = o;    o += RP * 4;
  L.lse_off = o;  o += RP * 4;
  L.total = o;
  return L;
}

// S (8 keys x all RP rows) = Q K^T; two independent accumulator chains.
template <int D, int MT>
__device__ __forceinline__ void qk8(float (&s)[MT][4], const __nv_bfloat16* Qs, const __nv_bfloat16* Kt, int n0,
                                    int lane) {
  constexpr int KROW = D + 8;
  float s2[MT][4];
#pragma unroll
  for (int mt = 0; mt < MT; ++mt)
#pragma unroll
    for (int i = 0; i < 4; ++i) s[mt][i] = s2[mt][i] = 0.f;
#pragma unroll
  for (int ks = 0; ks < D / 16; ks += 2) {
    unsigned b0, b1, b2, b3;
    ldsm_x4(b0, b1, b2, b3, Kt + (n0 + (lane & 7)) * KROW + ks * 16 + (lane >> 3) * 8);
#pragma unroll
    for (int mt = 0; mt < MT; ++mt) {
      unsigned a0, a1, a2, a3;
      const __nv_bfloat16* qa = Qs + (mt * 16 + (lane & 7) + ((lane >> 3) & 1) * 8) * KROW + (lane >> 4) * 8;
      ldsm_x4(a0, a1, a2, a3, qa + ks * 16);
      mma_bf16(s[mt], a0, a1, a2, a3, b0, b1);
      ldsm_x4(a0, a1, a2, a3, qa + (ks + 1) * 16);
      mma_bf16(s2[mt], a0, a1, a2, a3, b2, b3);
    }
  }
#pragma unroll
  for (int mt = 0; mt < MT; ++mt)
#pragma unroll
    for (int i = 0; i < 4; ++i) s[mt][i] += s2[mt][i];
}

// S (16 keys = two n8 tiles x all RP rows) = Q K^T.
template <int D, int MT>
__device__ __forceinline__ void qk16(float (&s)[MT][2][4], const __nv_bfloat16* Qs, const __nv_bfloat16* Kt,
                                     int k0, int lane) {
  constexpr int KROW = D + 8;
#pragma unroll
  for (int mt = 0; mt < MT; ++mt)
#pragma unroll
    for (int j = 0; j < 2; ++j)
#pragma unroll
      for (int i = 0; i < 4; ++i) s[mt][j][i] = 0.f;
#pragma unroll
  for (int ks = 0; ks < D / 16; ++ks) {
    unsigned b0, b1, b2, b3;  // (keys 0-7: d lo, d hi), (keys 8-15: d lo, d hi)
    ldsm_x4(b0, b1, b2, b3, Kt + (k0 + (lane & 7) + ((lane >> 4) << 3)) * KROW + ks * 16 + ((lane >> 3) & 1) * 8);
#pragma unroll
    for (int mt = 0; mt < MT; ++mt) {
      unsigned a0, a1, a2, a3;
      ldsm_x4(a0, a1, a2, a3,
              Qs + (mt * 16 + (lane & 7) + ((lane >> 3) & 1) * 8) * KROW + ks * 16 + (lane >> 4) * 8);
      mma_bf16(s[mt][0], a0, a1, a2, a3, b0, b1);
      mma_bf16(s[mt][1], a0, a1, a2, a3, b2, b3);
    }
  }
}

template <int D, int MT, int NSLOT>
__global__ void __launch_bounds__(NT, (MT <= 2 && NSLOT <= 4 ? 2 : 1)) attn_mma_kernel(const Params p) {
  constexpr int RP = MT * 16;
  constexpr int KROW = D + 8;
  constexpr int DCH = D / 8;       // 16-byte chunks per key row
  constexpr int NPAIR = NSLOT / 2;
  constexpr int TILE = TK * KROW;  // bf16 elements per ring slot
  constexpr int DH = D / 2;        // output columns per warp in pass 2
  constexpr int NTD = DH / 8;      // n8 tiles per warp in pass 2

  cg::cluster_group cluster = cg::this_cluster();
  const int C = static_cast<int>(cluster.num_blocks());
  const int crank = static_cast<int>(cluster.block_rank());
  const int h = blockIdx.y;
  const Item it = load_item(p.items, blockIdx.z);
  const int G = p.q_heads / p.kv.kv_heads;
  const int R = it.nq * G;
  const int Nk = it.num_keys();
  const int kb = crank * p.chunk;
  const int ke = min(Nk, kb + p.chunk);
  const int nk = max(0, ke - kb);
  const int ntiles = (nk + TK - 1) / TK;

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g4 = lane >> 2, t4 = lane & 3;

  extern __shared__ __align__(128) unsigned char smem[];
  const Layout L = make_layout(D, MT, NSLOT, p.chunk);
  __nv_bfloat16* ring = reinterpret_cast<__nv_bfloat16*>(smem + L.ring_off);
  __nv_bfloat16* Qs = reinterpret_cast<__nv_bfloat16*>(smem + L.q_off);
  int32_t* spos = reinterpret_cast<int32_t*>(smem + L.pos_off);
  int32_t* sslot = reinterpret_cast<int32_t*>(smem + L.slot_off);
  float* wm = reinterpret_cast<float*>(smem + L.wm_off);
  float* wl = reinterpret_cast<float*>(smem + L.wl_off);
  float* rowm = reinterpret_cast<float*>(smem + L.m_off);
  float* rowl = reinterpret_cast<float*>(smem + L.l_off);
  float* rowlse = reinterpret_cast<float*>(smem + L.lse_off);

  const int kvh = p.kv.kv_heads;
  // per-head base: slot s of this head starts at (s * kvh) * D
  const __nv_bfloat16* Kg = static_cast<const __nv_bfloat16*>(p.kv.k) + (int64_t)p.layer * p.kv.layer_stride + h * D;
  const __nv_bfloat16* Vg = static_cast<const __nv_bfloat16*>(p.kv.v) + (int64_t)p.layer * p.kv.layer_stride + h * D;
  const uint64_t keep = policy_evict_last();
  const uint64_t drop = policy_evict_first();

  // ---- setup: key positions / slots of this chunk, query rows ----
  for (int j = tid; j < ntiles * TK; j += NT) {
    const int gj = kb + j;
    int pos = 0x7fffffff, slot = -1;
    if (gj < ke) {
      pos = it.key_pos(p.crit, gj);
      slot = static_cast<int>(p.kv.slot_of(it.table_row, pos));
    }
    spos[j] = pos;
    sslot[j] = slot;
  }
  for (int i = tid; i < RP * DCH; i += NT) {
    const int r = i / DCH, c = i - r * DCH;
    uint4 v = make_uint4(0, 0, 0, 0);
    if (r < R) {
      const int qt = r / G, g = r - qt * G;
      v = *reinterpret_cast<const uint4*>(p.q + ((int64_t)(it.q_row0 + qt) * p.q_heads + h * G + g) * D + c * 8);
    }
    *reinterpret_cast<uint4*>(Qs + r * KROW + c * 8) = v;
  }
  __syncthreads();

  // one tile (64 keys) into a ring slot; thread -> 4 coalesced 16-byte chunks
  auto load_tile = [&](const __nv_bfloat16* base, int t, __nv_bfloat16* dst, uint64_t pol) {
#pragma unroll
    for (int i = tid; i < TK * DCH; i += NT) {
      const int kk = i / DCH, c = i - kk * DCH;
      const int slot = sslot[t * TK + kk];
      cp_async16(dst + kk * KROW + c * 8, base + (int64_t)(slot < 0 ? 0 : slot) * (kvh * D) + c * 8,
                 slot < 0 ? 0 : 16, pol);
    }
  };
  // every key of tile t exists, precedes every query row, and no planted bias
  auto tile_full = [&](int t) -> bool {
    if (p.n_planted != 0) return false;
    const int last = t * TK + TK - 1;
    return kb + last < ke && (kb + last < it.crit_len || spos[last] <= it.qpos0);
  };
  auto visible = [&](int jl, int r) -> bool {
    const int gj = kb + jl;
    return gj < ke && r < R && (gj < it.crit_len || spos[jl] <= it.qpos0 + r / G);
  };
  auto bias_of = [&](int jl) -> float {
    return p.n_planted ? planted_bias(p.planted, p.n_planted, p.bonus_log2, spos[jl]) : 0.f;
  };

  // ================= pass 1: row statistics =================
  float pm[MT][2], pl[MT][2];
#pragma unroll
  for (int mt = 0; mt < MT; ++mt) pm[mt][0] = pm[mt][1] = -INFINITY, pl[mt][0] = pl[mt][1] = 0.f;
  {
    const int n0 = warp * 8;
#pragma unroll
    for (int s = 0; s < NSLOT - 1; ++s) {
      if (s < ntiles) load_tile(Kg, s, ring + s * TILE, keep);
      cp_async_commit();
    }
    for (int t = 0; t < ntiles; ++t) {
      cp_async_wait<NSLOT - 2>();
      __syncthreads();
      {
        const int nt = t + NSLOT - 1;
        if (nt < ntiles) load_tile(Kg, nt, ring + (nt % NSLOT) * TILE, keep);
        cp_async_commit();
      }
      float sacc[MT][4];
      qk8<D, MT>(sacc, Qs, ring + (t % NSLOT) * TILE, n0, lane);
      if (tile_full(t)) {
#pragma unroll
        for (int mt = 0; mt < MT; ++mt)
#pragma unroll
          for (int hh = 0; hh < 2; ++hh) {
            const float s0 = sacc[mt][hh * 2] * p.scale_log2, s1 = sacc[mt][hh * 2 + 1] * p.scale_log2;
            const float nm = fmaxf(pm[mt][hh], fmaxf(s0, s1));
            pl[mt][hh] = pl[mt][hh] * exp2f(pm[mt][hh] - nm) + exp2f(s0 - nm) + exp2f(s1 - nm);
            pm[mt][hh] = nm;
          }
      } else {
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int jl = t * TK + n0 + 2 * t4 + e;
          const float bias = bias_of(jl);
#pragma unroll
          for (int mt = 0; mt < MT; ++mt)
#pragma unroll
            for (int hh = 0; hh < 2; ++hh) {
              if (visible(jl, mt * 16 + g4 + hh * 8)) {
                const float s = fmaf(sacc[mt][hh * 2 + e], p.scale_log2, bias);
                const float nm = fmaxf(pm[mt][hh], s);
                pl[mt][hh] = pl[mt][hh] * exp2f(pm[mt][hh] - nm) + exp2f(s - nm);
                pm[mt][hh] = nm;
              }
            }
        }
      }
    }
  }
  cp_async_wait<0>();
  // combine the 4 lanes sharing a row, then the 8 warps
#pragma unroll
  for (int mt = 0; mt < MT; ++mt)
#pragma unroll
    for (int hh = 0; hh < 2; ++hh) {
      float m = pm[mt][hh], l = pl[mt][hh];
#pragma unroll
      for (int o = 1; o <= 2; o <<= 1) {
        const float om = __shfl_xor_sync(0xffffffffu, m, o);
        const float ol = __shfl_xor_sync(0xffffffffu, l, o);
        const float nm = fmaxf(m, om);
        l = (nm == -INFINITY) ? 0.f : l * exp2f(m - nm) + ol * exp2f(om - nm);
        m = nm;
      }
      if (t4 == 0) {
        wm[warp * RP + mt * 16 + g4 + hh * 8] = m;
        wl[warp * RP + mt * 16 + g4 + hh * 8] = l;
      }
    }
  __syncthreads();
  // prefetch the first K/V pairs of pass 2 while statistics are exchanged
#pragma unroll
  for (int s = 0; s < NPAIR - 1; ++s) {
    if (s < ntiles) {
      load_tile(Kg, s, ring + (2 * s) * TILE, drop);
      load_tile(Vg, s, ring + (2 * s + 1) * TILE, drop);
    }
    cp_async_commit();
  }
  if (tid < RP) {
    float m = -INFINITY, l = 0.f;
    for (int w = 0; w < NW; ++w) {
      const float om = wm[w * RP + tid], ol = wl[w * RP + tid];
      const float nm = fmaxf(m, om);
      l = (nm == -INFINITY) ? 0.f : l * exp2f(m - nm) + ol * exp2f(om - nm);
      m = nm;
    }
    rowm[tid] = m;
    rowl[tid] = l;
  }
  cluster.sync();
  // ---- exact log-sum-exp over the cluster (DSMEM) ----
  if (tid < RP) {
    float lse2 = INFINITY;  // padding rows -> P = 0
    if (tid < R) {
      float M = -INFINITY;
      for (int c = 0; c < C; ++c) M = fmaxf(M, *cluster.map_shared_rank(rowm + tid, c));
      float Ls = 0.f;
      for (int c = 0; c < C; ++c) {
        const float mc = *cluster.map_shared_rank(rowm + tid, c);
        if (mc != -INFINITY) Ls += *cluster.map_shared_rank(rowl + tid, c) * exp2f(mc - M);
      }
      lse2 = M + log2f(Ls);
    }
    rowlse[tid] = lse2;
  }
  __syncthreads();

  // ================= pass 2: P (registers), scores, O = P V =================
  const int kg = warp & 3;   // 16-key group of the tile
  const int dh = warp >> 2;  // output-column half
  const int k0 = kg * 16;
  const bool scores = p.acc != nullptr && it.acc_row >= 0 && dh == 0;
  float lse_r[MT][2];
#pragma unroll
  for (int mt = 0; mt < MT; ++mt) lse_r[mt][0] = rowlse[mt * 16 + g4], lse_r[mt][1] = rowlse[mt * 16 + g4 + 8];
  float oacc[MT][NTD][4];
#pragma unroll
  for (int mt = 0; mt < MT; ++mt)
#pragma unroll
    for (int nt = 0; nt < NTD; ++nt) oacc[mt][nt][0] = oacc[mt][nt][1] = oacc[mt][nt][2] = oacc[mt][nt][3] = 0.f;

  for (int t = 0; t < ntiles; ++t) {
    cp_async_wait<NPAIR - 2>();
    __syncthreads();
    {
      const int nt = t + NPAIR - 1;
      if (nt < ntiles) {
        load_tile(Kg, nt, ring + (2 * (nt % NPAIR)) * TILE, drop);
        load_tile(Vg, nt, ring + (2 * (nt % NPAIR) + 1) * TILE, drop);
      }
      cp_async_commit();
    }
    const __nv_bfloat16* Kt = ring + (2 * (t % NPAIR)) * TILE;
    const __nv_bfloat16* Vt = ring + (2 * (t % NPAIR) + 1) * TILE;
    float sacc[MT][2][4];  // [mt][n8 tile j][c0..c3]
    qk16<D, MT>(sacc, Qs, Kt, k0, lane);
    const bool full = tile_full(t);
#pragma unroll
    for (int j = 0; j < 2; ++j)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int jl = t * TK + k0 + j * 8 + 2 * t4 + e;
        const float bias = full ? 0.f : bias_of(jl);
#pragma unroll
        for (int mt = 0; mt < MT; ++mt)
#pragma unroll
          for (int hh = 0; hh < 2; ++hh) {
            const bool vis = full || visible(jl, mt * 16 + g4 + hh * 8);
            sacc[mt][j][hh * 2 + e] =
                vis ? exp2f(fmaf(sacc[mt][j][hh * 2 + e], p.scale_log2, bias) - lse_r[mt][hh]) : 0.f;
          }
      }
    // PillarAttn scores: sum the G rows of each query token (lanes g4 .. g4+G-1)
    if (scores) {
      const int gl = min(G, 8);
#pragma unroll
      for (int mt = 0; mt < MT; ++mt)
#pragma unroll
        for (int j = 0; j < 2; ++j)
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            float v0 = sacc[mt][j][e], v1 = sacc[mt][j][2 + e];
            if (G >= 16) v0 += v1;
            for (int o = 4; o < 4 * gl; o <<= 1) {
              v0 += __shfl_xor_sync(0xffffffffu, v0, o);
              v1 += __shfl_xor_sync(0xffffffffu, v1, o);
            }
            const int jl = t * TK + k0 + j * 8 + 2 * t4 + e;
            if (kb + jl < ke && (g4 % gl) == 0) {
              const int pos = spos[jl];
              const int tok0 = (mt * 16 + g4) / G;
              if (v0 != 0.f && tok0 < it.nq)
                atomicAdd(p.acc + (int64_t)(it.acc_row + tok0 * it.acc_step) * p.acc_stride + pos, v0);
              if (G < 16) {
                const int tok1 = (mt * 16 + g4 + 8) / G;
                if (v1 != 0.f && tok1 < it.nq)
                  atomicAdd(p.acc + (int64_t)(it.acc_row + tok1 * it.acc_step) * p.acc_stride + pos, v1);
              }
            }
          }
    }
    // O += P V over this warp's 16 keys and DH columns; P's C fragments are
    // the A fragments of the k16 step (rows g4/g4+8, keys 2t4.. of each n8 tile)
    unsigned a[MT][4];
#pragma unroll
    for (int mt = 0; mt < MT; ++mt) {
      a[mt][0] = pack_bf16(sacc[mt][0][0], sacc[mt][0][1]);
      a[mt][1] = pack_bf16(sacc[mt][0][2], sacc[mt][0][3]);
      a[mt][2] = pack_bf16(sacc[mt][1][0], sacc[mt][1][1]);
      a[mt][3] = pack_bf16(sacc[mt][1][2], sacc[mt][1][3]);
    }
#pragma unroll
    for (int nt = 0; nt < NTD; nt += 2) {
      unsigned b0, b1, b2, b3;
      ldsm_x4_t(b0, b1, b2, b3,
                Vt + (k0 + (lane & 7) + ((lane >> 3) & 1) * 8) * KROW + dh * DH + nt * 8 + (lane >> 4) * 8);
#pragma unroll
      for (int mt = 0; mt < MT; ++mt) {
        mma_bf16(oacc[mt][nt], a[mt][0], a[mt][1], a[mt][2], a[mt][3], b0, b1);
        mma_bf16(oacc[mt][nt + 1], a[mt][0], a[mt][1], a[mt][2], a[mt][3], b2, b3);
      }
    }
  }
  cp_async_wait<0>();
  __syncthreads();

  // ---- O partials: 4 key groups -> smem (ring reused), then cluster DSMEM reduce ----
  float* Ob = reinterpret_cast<float*>(ring);  // [RP][D]
  for (int i = tid; i < RP * D; i += NT) Ob[i] = 0.f;
  __syncthreads();
#pragma unroll
  for (int mt = 0; mt < MT; ++mt)
#pragma unroll
    for (int nt = 0; nt < NTD; ++nt)
#pragma unroll
      for (int hh = 0; hh < 2; ++hh) {
        float* dst = Ob + (mt * 16 + g4 + hh * 8) * D + dh * DH + nt * 8 + 2 * t4;
        atomicAdd(dst, oacc[mt][nt][hh * 2]);
        atomicAdd(dst + 1, oacc[mt][nt][hh * 2 + 1]);
      }
  cluster.sync();
  {
    const int mine = (R - crank + C - 1) / C;  // rows r = crank + i*C
    for (int i = tid; i < mine * (D / 4); i += NT) {
      const int ri = i / (D / 4), c4 = i - ri * (D / 4);
      const int r = crank + ri * C;
      float4 s = make_float4(0.f, 0.f, 0.f, 0.f);
      for (int c = 0; c < C; ++c) {
        const float4 v = *reinterpret_cast<const float4*>(cluster.map_shared_rank(Ob + r * D + c4 * 4, c));
        s.x += v.x; s.y += v.y; s.z += v.z; s.w += v.w;
      }
      const int qt = r / G, g = r - qt * G;
      __nv_bfloat162* dst = reinterpret_cast<__nv_bfloat162*>(
          p.out + ((int64_t)(it.q_row0 + qt) * p.q_heads + h * G + g) * D + c4 * 4);
      dst[0] = __floats2bfloat162_rn(s.x, s.y);
      dst[1] = __floats2bfloat162_rn(s.z, s.w);
    }
    if (p.lse_out != nullptr && crank == 0 && tid < R) {
      const int qt = tid / G, g = tid - qt * G;
      p.lse_out[(int64_t)(it.q_row0 + qt) * p.q_heads + h * G + g] = rowlse[tid] * LN2;
    }
  }
  cluster.sync();
}

template <int D, int MT, int NSLOT>
int launch_one(const Params& prm, int C, int num_items, int kv_heads, cudaStream_t stream) {
  auto kern = attn_mma_kernel<D, MT, NSLOT>;
  const int smem = make_layout(D, MT, NSLOT, prm.chunk).total;
  static int configured = 0;
  if (smem > configured) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    configured = smem;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(C, kv_heads, num_items);
  cfg.blockDim = dim3(NT);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = C;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaError_t e = cudaLaunchKernelEx(&cfg, kern, prm);
  count_launch();
  if (e != cudaSuccess) {
    set_error(std::string("sd_attention launch: ") + cudaGetErrorString(e));
    return (int)e;
  }
  return 0;
}

}  // namespace mma_attn

bool mma_attn_supported(int dtype, int D, int rows) {
  return dtype == SD_DTYPE_BF16 && (D == 64 || D == 128) && rows >= 1 && rows <= 80;
}

// Cluster size: enough CTAs for ~4 waves of 2 CTAs/SM, chunks of at most
// ~512 keys so the K re-read of pass 2 stays L2-resident, C <= 16.
static int env_int(const char* name, int dflt) {
  const char* v = getenv(name);
  return v && *v ? atoi(v) : dflt;
}

// Ring depth (tiles of 64 keys in shared memory): 4 -> two CTAs per SM,
// 10 -> one CTA per SM with ~9 K tiles / 4 K+V pairs in flight.
static int ring_slots() {
  static const int n = env_int("SD_ATTN_NSLOT", 10);
  return n;
}

// Cluster size C: enough CTAs for the machine, chunks of at most
// SD_ATTN_CHUNK_TILES tiles so the K re-read of pass 2 stays L2-resident,
// C <= 16 (non-portable cluster sizes are enabled); SD_ATTN_C forces C.
static void plan_mma(int max_keys, int num_items, int kv_heads, int* C_out, int* chunk_out) {
  using namespace mma_attn;
  const int tiles = (max_keys + TK - 1) / TK;
  const int work = num_items * kv_heads;
  const int per_sm = ring_slots() <= 4 ? 2 : 1;
  static const int max_chunk_tiles = env_int("SD_ATTN_CHUNK_TILES", 16);
  static const int force_c = env_int("SD_ATTN_C", 0);
  int c = (2 * per_sm * 148 + work - 1) / work;  // parallelism target (~2 waves)
  const int c_l2 = (tiles + max_chunk_tiles - 1) / max_chunk_tiles;
  if (c_l2 > c) c = c_l2;
  if (force_c > 0) c = force_c;
  if (c > tiles) c = tiles;
  if (c > 16) c = 16;
  if (c < 1) c = 1;
  *C_out = c;
  *chunk_out = ((tiles + c - 1) / c) * TK;
}

bool mma_attn_plannable(int dtype, int D, int rows, int max_keys, int num_items, int kv_heads) {
  (void)max_keys;
  (void)num_items;
  (void)kv_heads;
  return mma_attn_supported(dtype, D, rows);
}

int launch_attn_mma(const void* q, void* out, float* lse, const sd_paged_kv* kvp, int layer,
                    const int32_t* items, int num_items, int max_keys, int max_nq, const int32_t* crit,
                    float* acc, int64_t acc_stride, const int32_t* planted, int n_planted, float bonus,
                    int q_heads, float scale, cudaStream_t stream, bool* handled) {
  using namespace mma_attn;
  const int D = kvp->head_dim;
  const int G = q_heads / kvp->kv_heads;
  const int rows = max_nq * G;
  *handled = false;
  if (!mma_attn_supported(kvp->dtype, D, rows)) return 0;
  const int MT = (rows + 15) / 16;
  int C = 1, chunk = TK;
  plan_mma(max_keys < 1 ? 1 : max_keys, num_items, kvp->kv_heads, &C, &chunk);
  Params prm;
  prm.q = static_cast<const __nv_bfloat16*>(q);
  prm.out = static_cast<__nv_bfloat16*>(out);
  prm.lse_out = lse;
  prm.kv = make_paged(kvp);
  prm.layer = layer;
  prm.items = items;
  prm.crit = crit;
  prm.acc = acc;
  prm.acc_stride = acc_stride;
  prm.planted = planted;
  prm.n_planted = n_planted;
  prm.bonus_log2 = bonus * LOG2E;
  prm.q_heads = q_heads;
  prm.scale_log2 = scale * LOG2E;
  prm.chunk = chunk;
  *handled = true;
  const int nslot = ring_slots();
#define SD_MMA_CASE(DD, M)                                                                       \
  if (D == DD && MT == M) {                                                                      \
    if (nslot <= 4) return launch_one<DD, M, 4>(prm, C, num_items, kvp->kv_heads, stream);       \
    return launch_one<DD, M, 10>(prm, C, num_items, kvp->kv_heads, stream);                      \
  }
  SD_MMA_CASE(128, 1) SD_MMA_CASE(128, 2) SD_MMA_CASE(128, 3) SD_MMA_CASE(128, 4) SD_MMA_CASE(128, 5)
  SD_MMA_CASE(64, 1) SD_MMA_CASE(64, 2) SD_MMA_CASE(64, 3) SD_MMA_CASE(64, 4) SD_MMA_CASE(64, 5)
#undef SD_MMA_CASE
  *handled = false;
  return 0;
}

}  // namespace sd
