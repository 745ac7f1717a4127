// Warp-specialized paged attention for sm_100a (K1 sparse draft + K2 verify
// with PillarAttn score emission).  Same math and cluster decomposition as
// attn_mma.cu, different execution model:
//
//   warp 8 (producer)  streams 256-byte K / V key rows HBM -> a shared-memory
//                      ring with cp.async.bulk (TMA engine, one instruction per
//                      key row, 2 per lane per 64-key tile), completion tracked
//                      by per-slot mbarriers (expect_tx); waits on per-slot
//                      "empty" mbarriers before reusing a slot.  It runs ahead
//                      of the consumers across the pass boundary, so pass-2
//                      tiles are already in flight during the cluster exchange.
//   warps 0-7 (math)   never execute a CTA-wide barrier in the tile loops:
//                      wait "full[slot]" -> mma.sync (bf16, fp32 accumulate)
//                      -> softmax / scores -> arrive "empty[slot]".
//
// Fill sequence per CTA: pass 1 K(0..T-1), pass 2 K(0),V(0),K(1),V(1),...
// Fill f lives in slot f % NSLOT with mbarrier phase (f / NSLOT) & 1.
//
// Rows: verify items (1 < nq <= 8) use GROUP-major rows r = g*8 + token so a
// thread's C-fragment rows (g4, g4+8, g4+16, ...) are all heads of ONE token:
// the PillarAttn score sum over the GQA group is register-local (no
// shuffles).  Drafts / prefill chunks use token-major rows r = token*G + g.
//
// Restates model.py:229-253 (_attend) for forward_full (model.py:318-334) and
// forward_sparse (model.py:360-380), and the score path selection.py:78-135.
#include <cooperative_groups.h>

#include "common.cuh"

namespace cg = cooperative_groups;

namespace sd {
namespace ws_attn {

constexpr int TK = 64;      // keys per tile
constexpr int NCW = 8;      // math warps
constexpr int NT = (NCW + 1) * 32;
constexpr float LOG2E = 1.4426950408889634f;
constexpr float LN2 = 0.6931471805599453f;

// ---- PTX helpers ---------------------------------------------------------------------
__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_arrive_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_copy(void* dst, const void* src, unsigned bytes, uint64_t* bar,
                                          uint64_t policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;\n" ::
          "r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}
__device__ __forceinline__ void cp_async16_pol(void* dst, const void* src, uint64_t policy) {
  asm volatile("cp.async.cg.shared.global.L2::cache_hint [%0], [%1], 16, %2;\n" ::"r"(smem_u32(dst)), "l"(src),
               "l"(policy)
               : "memory");
}
__device__ __forceinline__ void cp_async_mbar_arrive(uint64_t* bar) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}
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
__device__ __forceinline__ void cluster_arrive() { asm volatile("barrier.cluster.arrive.release.aligned;\n" ::: "memory"); }
__device__ __forceinline__ void cluster_wait() { asm volatile("barrier.cluster.wait.acquire.aligned;\n" ::: "memory"); }
__device__ __forceinline__ void math_bar() { asm volatile("bar.sync 1, %0;\n" ::"n"(NCW * 32) : "memory"); }

__device__ __forceinline__ void ldsm_x4(unsigned& r0, unsigned& r1, unsigned& r2, unsigned& r3, const void* p) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];\n"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3) : "r"(smem_u32(p)));
}
__device__ __forceinline__ void ldsm_x4_t(unsigned& r0, unsigned& r1, unsigned& r2, unsigned& r3, const void* p) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];\n"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3) : "r"(smem_u32(p)));
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
__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;\n" : "=f"(y) : "f"(x));
  return y;
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
  int nomath; // diagnostics: stream the tiles, skip the math (SD_ATTN_NOMATH=1)
  int loader; // 0 = cp.async.bulk per key row, 1 = 16-byte cp.async + mbarrier arrive
};

struct Layout {
  int bar_off, ring_off, q_off, pos_off, slot_off, wm_off, wl_off, m_off, l_off, lse_off, total;
};
__host__ __device__ inline Layout make_layout(int D, int MT, int nslot, int chunk) {
  const int RP = MT * 16;
  const int krow = D + 8;
  Layout L;
  int o = 0;
  L.bar_off = o;  o += 2 * nslot * 8;
  o = (o + 127) & ~127;
  L.ring_off = o;
  {
    const int ring = nslot * TK * krow * 2;
    const int obuf = RP * D * 4;
    o += ring > obuf ? ring : obuf;
  }
  L.q_off = o;    o += RP * krow * 2;
  L.pos_off = o;  o += chunk * 4;
  L.slot_off = o; o += chunk * 4;
  L.wm_off = o;   o += NCW * RP * 4;
  L.wl_off = o;   o += NCW * RP * 4;
  L.m_off = o;    o += RP * 4;
  L.l_off = o;    o += RP * 4;
  L.lse_off = o;  o += RP * 4;
  L.total = o;
  return L;
}

// S (8 keys x all RP rows) = Q K^T, two independent accumulator chains.
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
    unsigned b0, b1, b2, b3;
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

template <int D, int MT, int NSLOT, bool GM>
__global__ void __launch_bounds__(NT, (MT <= 2 && NSLOT <= 5) ? 2 : 1) attn_ws_kernel(const Params p) {
  constexpr int RP = MT * 16;
  constexpr int KROW = D + 8;
  constexpr int DCH = D / 8;
  constexpr int TILE = TK * KROW;
  constexpr int DH = D / 2;
  constexpr int NTD = DH / 8;
  constexpr unsigned ROWB = D * 2;  // bytes per key row

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
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + L.bar_off);
  uint64_t* empty = full + NSLOT;
  __nv_bfloat16* ring = reinterpret_cast<__nv_bfloat16*>(smem + L.ring_off);
  __nv_bfloat16* Qs = reinterpret_cast<__nv_bfloat16*>(smem + L.q_off);
  int32_t* spos = reinterpret_cast<int32_t*>(smem + L.pos_off);
  int32_t* sslot = reinterpret_cast<int32_t*>(smem + L.slot_off);
  float* wm = reinterpret_cast<float*>(smem + L.wm_off);
  float* wl = reinterpret_cast<float*>(smem + L.wl_off);
  float* rowm = reinterpret_cast<float*>(smem + L.m_off);
  float* rowl = reinterpret_cast<float*>(smem + L.l_off);
  float* rowlse = reinterpret_cast<float*>(smem + L.lse_off);

  // row r -> (token, group member)
  auto row_tok = [&](int r) { return GM ? (r & 7) : r / G; };
  auto row_g = [&](int r) { return GM ? (r >> 3) : r % G; };
  auto row_real = [&](int r) { return GM ? ((r & 7) < it.nq && (r >> 3) < G) : r < R; };

  // ---- setup (all warps) ----
  if (tid < NSLOT) {
    mbar_init(full + tid, p.loader == 0 ? 1 : 32);
    mbar_init(empty + tid, NCW);
  }
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
    if (row_real(r)) {
      v = *reinterpret_cast<const uint4*>(
          p.q + ((int64_t)(it.q_row0 + row_tok(r)) * p.q_heads + h * G + row_g(r)) * D + c * 8);
    }
    *reinterpret_cast<uint4*>(Qs + r * KROW + c * 8) = v;
  }
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  __syncthreads();

  const int kvh = p.kv.kv_heads;
  const __nv_bfloat16* Kg = static_cast<const __nv_bfloat16*>(p.kv.k) + (int64_t)p.layer * p.kv.layer_stride + h * D;
  const __nv_bfloat16* Vg = static_cast<const __nv_bfloat16*>(p.kv.v) + (int64_t)p.layer * p.kv.layer_stride + h * D;

  if (warp == NCW) {
    // ===================== producer warp =====================
    const uint64_t keep = policy_evict_last();
    const uint64_t drop = policy_evict_first();
    const int total = 3 * ntiles;
    const int last_valid = nk - 1;
    for (int f = 0; f < total; ++f) {
      const int s = f % NSLOT;
      if (f >= NSLOT) mbar_wait(empty + s, ((f / NSLOT) - 1) & 1);
      int t;
      const __nv_bfloat16* base;
      uint64_t pol;
      if (f < ntiles) {
        t = f, base = Kg, pol = keep;
      } else {
        const int g2 = f - ntiles;
        t = g2 >> 1;
        base = (g2 & 1) ? Vg : Kg;
        pol = drop;
      }
      __nv_bfloat16* dst = ring + s * TILE;
      if (p.loader == 0) {
        // one bulk async copy (TMA engine) per 256-byte key row
        if (lane == 0) mbar_arrive_tx(full + s, TK * ROWB);
        __syncwarp();
#pragma unroll
        for (int kk = lane; kk < TK; kk += 32) {
          int j = t * TK + kk;
          if (j > last_valid) j = last_valid;  // duplicate a valid row; masked by the math warps
          bulk_copy(dst + kk * KROW, base + (int64_t)sslot[j] * (kvh * D), ROWB, full + s, pol);
        }
      } else {
        // 16-byte cp.async (LDGSTS), 32 / DCH key rows per warp instruction
        // (coalesced), then an mbarrier arrive that fires when this lane's
        // copies land.  The tile's 64 slots are read once (2 per lane) and
        // broadcast with shuffles, so no load sits on the issue path.
        const int j0 = min(t * TK + lane, last_valid), j1 = min(t * TK + lane + 32, last_valid);
        const int slot0 = sslot[j0], slot1 = sslot[j1];
        constexpr int KPI = 32 / DCH;  // key rows per warp instruction
        const int sub = lane / DCH, c = lane - sub * DCH;
#pragma unroll 8
        for (int m = 0; m < TK / KPI; ++m) {
          const int kk = m * KPI + sub;  // key of this lane in instruction m
          const int src_lane = kk & 31;
          const int sa = __shfl_sync(0xffffffffu, slot0, src_lane);
          const int sb = __shfl_sync(0xffffffffu, slot1, src_lane);
          const int slot = kk < 32 ? sa : sb;
          cp_async16_pol(dst + kk * KROW + c * 8, base + (int64_t)slot * (kvh * D) + c * 8, pol);
        }
        cp_async_mbar_arrive(full + s);
      }
      if (f == ntiles - 1) cluster_arrive();  // pass-1 fills issued: let the exchange proceed
    }
    if (ntiles == 0) cluster_arrive();
    cluster_wait();   // exchange barrier
    cluster_arrive();  // O-partials barrier
    cluster_wait();
    cluster_arrive();  // exit guard
    cluster_wait();
    return;
  }

  // ===================== math warps =====================
  auto tile_full = [&](int t) -> bool {
    if (p.n_planted != 0) return false;
    const int last = t * TK + TK - 1;
    return kb + last < ke && (kb + last < it.crit_len || spos[last] <= it.qpos0);
  };
  auto visible = [&](int jl, int r) -> bool {
    const int gj = kb + jl;
    return gj < ke && row_real(r) && (gj < it.crit_len || spos[jl] <= it.qpos0 + row_tok(r));
  };
  auto bias_of = [&](int jl) -> float {
    return p.n_planted ? planted_bias(p.planted, p.n_planted, p.bonus_log2, spos[jl]) : 0.f;
  };

  // ---- pass 1: row statistics ----
  float pm[MT][2], pl[MT][2];
#pragma unroll
  for (int mt = 0; mt < MT; ++mt) pm[mt][0] = pm[mt][1] = -INFINITY, pl[mt][0] = pl[mt][1] = 0.f;
  {
    const int n0 = warp * 8;
    for (int t = 0; t < ntiles; ++t) {
      const int s = t % NSLOT;
      mbar_wait(full + s, (t / NSLOT) & 1);
      if (p.nomath) {
        __syncwarp();
        if (lane == 0) mbar_arrive(empty + s);
        continue;
      }
      float sacc[MT][4];
      qk8<D, MT>(sacc, Qs, ring + s * TILE, n0, lane);
      __syncwarp();
      if (lane == 0) mbar_arrive(empty + s);
      if (tile_full(t)) {
#pragma unroll
        for (int mt = 0; mt < MT; ++mt)
#pragma unroll
          for (int hh = 0; hh < 2; ++hh) {
            const float s0 = sacc[mt][hh * 2] * p.scale_log2, s1 = sacc[mt][hh * 2 + 1] * p.scale_log2;
            const float nm = fmaxf(pm[mt][hh], fmaxf(s0, s1));
            pl[mt][hh] = pl[mt][hh] * ex2(pm[mt][hh] - nm) + ex2(s0 - nm) + ex2(s1 - nm);
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
                pl[mt][hh] = pl[mt][hh] * ex2(pm[mt][hh] - nm) + ex2(s - nm);
                pm[mt][hh] = nm;
              }
            }
        }
      }
    }
  }
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
        l = (nm == -INFINITY) ? 0.f : l * ex2(m - nm) + ol * ex2(om - nm);
        m = nm;
      }
      if (t4 == 0) {
        wm[warp * RP + mt * 16 + g4 + hh * 8] = m;
        wl[warp * RP + mt * 16 + g4 + hh * 8] = l;
      }
    }
  math_bar();
  if (tid < RP) {
    float m = -INFINITY, l = 0.f;
    for (int w = 0; w < NCW; ++w) {
      const float om = wm[w * RP + tid], ol = wl[w * RP + tid];
      const float nm = fmaxf(m, om);
      l = (nm == -INFINITY) ? 0.f : l * ex2(m - nm) + ol * ex2(om - nm);
      m = nm;
    }
    rowm[tid] = m;
    rowl[tid] = l;
  }
  cluster_arrive();
  cluster_wait();
  if (tid < RP) {
    float lse2 = INFINITY;  // padding rows -> P = 0
    if (row_real(tid)) {
      float M = -INFINITY;
      for (int c = 0; c < C; ++c) M = fmaxf(M, *cluster.map_shared_rank(rowm + tid, c));
      float Ls = 0.f;
      for (int c = 0; c < C; ++c) {
        const float mc = *cluster.map_shared_rank(rowm + tid, c);
        if (mc != -INFINITY) Ls += *cluster.map_shared_rank(rowl + tid, c) * ex2(mc - M);
      }
      lse2 = M + log2f(Ls);
    }
    rowlse[tid] = lse2;
  }
  math_bar();

  // ---- pass 2: P in registers, scores, O = P V ----
  const int kg = warp & 3;
  const int dh = warp >> 2;
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
    const int fk = ntiles + 2 * t, fv = fk + 1;
    const int sk = fk % NSLOT, sv = fv % NSLOT;
    mbar_wait(full + sk, (fk / NSLOT) & 1);
    if (p.nomath) {
      __syncwarp();
      if (lane == 0) mbar_arrive(empty + sk);
      mbar_wait(full + sv, (fv / NSLOT) & 1);
      __syncwarp();
      if (lane == 0) mbar_arrive(empty + sv);
      continue;
    }
    float sacc[MT][2][4];
    qk16<D, MT>(sacc, Qs, ring + sk * TILE, k0, lane);
    __syncwarp();
    if (lane == 0) mbar_arrive(empty + sk);
    const bool fullt = tile_full(t);
#pragma unroll
    for (int j = 0; j < 2; ++j)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int jl = t * TK + k0 + j * 8 + 2 * t4 + e;
        const float bias = fullt ? 0.f : bias_of(jl);
#pragma unroll
        for (int mt = 0; mt < MT; ++mt)
#pragma unroll
          for (int hh = 0; hh < 2; ++hh) {
            const bool vis = fullt || visible(jl, mt * 16 + g4 + hh * 8);
            sacc[mt][j][hh * 2 + e] =
                vis ? ex2(fmaf(sacc[mt][j][hh * 2 + e], p.scale_log2, bias) - lse_r[mt][hh]) : 0.f;
          }
      }
    if (scores) {
      if constexpr (GM) {
        // this thread's rows g4 + 8*i are group members i of token g4
#pragma unroll
        for (int j = 0; j < 2; ++j)
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            float v = 0.f;
#pragma unroll
            for (int mt = 0; mt < MT; ++mt) v += sacc[mt][j][e] + sacc[mt][j][2 + e];
            const int jl = t * TK + k0 + j * 8 + 2 * t4 + e;
            if (g4 < it.nq && kb + jl < ke && v != 0.f)
              atomicAdd(p.acc + (int64_t)(it.acc_row + g4 * it.acc_step) * p.acc_stride + spos[jl], v);
          }
      } else {
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
    }
    unsigned a[MT][4];
#pragma unroll
    for (int mt = 0; mt < MT; ++mt) {
      a[mt][0] = pack_bf16(sacc[mt][0][0], sacc[mt][0][1]);
      a[mt][1] = pack_bf16(sacc[mt][0][2], sacc[mt][0][3]);
      a[mt][2] = pack_bf16(sacc[mt][1][0], sacc[mt][1][1]);
      a[mt][3] = pack_bf16(sacc[mt][1][2], sacc[mt][1][3]);
    }
    mbar_wait(full + sv, (fv / NSLOT) & 1);
    const __nv_bfloat16* Vt = ring + sv * TILE;
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
    __syncwarp();
    if (lane == 0) mbar_arrive(empty + sv);
  }

  // ---- O partials -> smem (ring reused once every fill is consumed) ----
  math_bar();
  float* Ob = reinterpret_cast<float*>(ring);  // [RP][D]
  for (int i = tid; i < RP * D; i += NCW * 32) Ob[i] = 0.f;
  math_bar();
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
  cluster_arrive();
  cluster_wait();
  {
    // rows of this CTA: r = crank + i*C over the RP padded rows, real rows only
    for (int i = tid; i < ((RP - crank + C - 1) / C) * (D / 4); i += NCW * 32) {
      const int ri = i / (D / 4), c4 = i - ri * (D / 4);
      const int r = crank + ri * C;
      if (!row_real(r)) continue;
      float4 s = make_float4(0.f, 0.f, 0.f, 0.f);
      for (int c = 0; c < C; ++c) {
        const float4 v = *reinterpret_cast<const float4*>(cluster.map_shared_rank(Ob + r * D + c4 * 4, c));
        s.x += v.x; s.y += v.y; s.z += v.z; s.w += v.w;
      }
      __nv_bfloat162* dst = reinterpret_cast<__nv_bfloat162*>(
          p.out + ((int64_t)(it.q_row0 + row_tok(r)) * p.q_heads + h * G + row_g(r)) * D + c4 * 4);
      dst[0] = __floats2bfloat162_rn(s.x, s.y);
      dst[1] = __floats2bfloat162_rn(s.z, s.w);
    }
    if (p.lse_out != nullptr && crank == 0 && tid < RP && row_real(tid))
      p.lse_out[(int64_t)(it.q_row0 + row_tok(tid)) * p.q_heads + h * G + row_g(tid)] = rowlse[tid] * LN2;
  }
  cluster_arrive();
  cluster_wait();
}

template <int D, int MT, int NSLOT, bool GM>
int launch_one(const Params& prm, int C, int num_items, int kv_heads, cudaStream_t stream) {
  auto kern = attn_ws_kernel<D, MT, NSLOT, GM>;
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
    set_error(std::string("sd_attention (ws) launch: ") + cudaGetErrorString(e));
    return (int)e;
  }
  return 0;
}

static int env_int(const char* name, int dflt) {
  const char* v = getenv(name);
  return v && *v ? atoi(v) : dflt;
}

}  // namespace ws_attn

// Cluster size: ~2 waves of CTAs, chunks <= SD_ATTN_CHUNK_TILES tiles (K re-read
// of pass 2 L2-resident), C <= 16; SD_ATTN_C forces C.
static void plan_ws(int max_keys, int num_items, int kv_heads, int per_sm, int* C_out, int* chunk_out) {
  using namespace ws_attn;
  const int tiles = (max_keys + TK - 1) / TK;
  const int work = num_items * kv_heads;
  static const int max_chunk_tiles = env_int("SD_ATTN_CHUNK_TILES", 16);
  static const int force_c = env_int("SD_ATTN_C", 0);
  int c = (2 * per_sm * 148 + work - 1) / work;
  const int c_l2 = (tiles + max_chunk_tiles - 1) / max_chunk_tiles;
  if (c_l2 > c) c = c_l2;
  if (force_c > 0) c = force_c;
  if (c > tiles) c = tiles;
  if (c > 16) c = 16;
  if (c < 1) c = 1;
  *C_out = c;
  *chunk_out = ((tiles + c - 1) / c) * TK;
}

int launch_attn_ws(const void* q, void* out, float* lse, const sd_paged_kv* kvp, int layer, const int32_t* items,
                   int num_items, int max_keys, int max_nq, const int32_t* crit, float* acc, int64_t acc_stride,
                   const int32_t* planted, int n_planted, float bonus, int q_heads, float scale, cudaStream_t stream,
                   bool* handled) {
  using namespace ws_attn;
  const int D = kvp->head_dim;
  const int G = q_heads / kvp->kv_heads;
  *handled = false;
  if (kvp->dtype != SD_DTYPE_BF16 || !(D == 64 || D == 128)) return 0;
  // group-major rows for verify-sized items (2..8 tokens, G <= 8); token-major otherwise
  const bool gm = max_nq >= 2 && max_nq <= 8 && G <= 8 && (G & (G - 1)) == 0 && G >= 2;
  const int rows = gm ? 8 * G : max_nq * G;
  if (rows > 80) return 0;
  const int MT = (rows + 15) / 16;
  static const int nslot_env = env_int("SD_ATTN_NSLOT", 5);
  const int nslot = nslot_env <= 5 ? 5 : 10;
  const int per_sm = (MT <= 2 && nslot <= 5) ? 2 : 1;
  int C = 1, chunk = TK;
  plan_ws(max_keys < 1 ? 1 : max_keys, num_items, kvp->kv_heads, per_sm, &C, &chunk);
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
  static const int nomath = env_int("SD_ATTN_NOMATH", 0);
  prm.nomath = nomath;
  static const int loader = env_int("SD_ATTN_LOADER", 1);
  prm.loader = loader;
  *handled = true;
#define SD_WS_CASE(DD, M)                                                                                    \
  if (D == DD && MT == M) {                                                                                  \
    if (gm) {                                                                                                \
      if (nslot == 5) return launch_one<DD, M, 5, true>(prm, C, num_items, kvp->kv_heads, stream);           \
      return launch_one<DD, M, 10, true>(prm, C, num_items, kvp->kv_heads, stream);                          \
    }                                                                                                        \
    if (nslot == 5) return launch_one<DD, M, 5, false>(prm, C, num_items, kvp->kv_heads, stream);            \
    return launch_one<DD, M, 10, false>(prm, C, num_items, kvp->kv_heads, stream);                           \
  }
  SD_WS_CASE(128, 1) SD_WS_CASE(128, 2) SD_WS_CASE(128, 3) SD_WS_CASE(128, 4) SD_WS_CASE(128, 5)
  SD_WS_CASE(64, 1) SD_WS_CASE(64, 2) SD_WS_CASE(64, 3) SD_WS_CASE(64, 4) SD_WS_CASE(64, 5)
#undef SD_WS_CASE
  *handled = false;
  return 0;
}

}  // namespace sd
