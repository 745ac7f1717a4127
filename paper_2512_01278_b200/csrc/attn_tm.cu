// TMEM-resident-logit paged attention for sm_100a: K1 sparse draft and K2
// verify with PillarAttn score emission, reading every K and V row from HBM
// exactly once.
//
// Why: the exact scores need each row's FINAL lse before exp(s - lse) can be
// summed over the GQA group, so the logits must survive until the cluster
// has reduced its (max, sum) statistics.  Re-reading K from L2 caps the SM
// load path at ~4.2 TB/s (tools/stream_probe.cu); shared memory is needed for
// the copy ring.  Blackwell's 256 KB of tensor memory per SM holds them
// instead: tcgen05.st after QK^T, tcgen05.ld before exp, no HBM, no smem.
//
//   grid = (C, kv_heads, items), cluster (C,1,1); CTA c owns keys
//   [c*chunk, (c+1)*chunk) of the item's key list (critical list, then the
//   dense causal range); one CTA per SM (512 TMEM columns, 10-slot ring).
//
//   warp 8 (producer)  16-byte cp.async (LDGSTS) of 256-byte key rows into a
//                      10 x 17 KB ring, completion on per-slot mbarriers;
//                      K tiles 0..T-1 then V tiles 0..T-1 (each row once).
//   warps 0-7 (math)   phase 1: S = Q K^T (mma.sync bf16 -> fp32), scale,
//                      causal mask, planted bias, online (max, sum), S -> TMEM.
//                      exchange: (max, sum) over the cluster via DSMEM -> lse.
//                      phase 2: S <- TMEM, P = exp2(S - lse) (final), scores
//                      acc[token][pos] += sum_g P (register-local: group-major
//                      rows), O += P V (mma.sync), DSMEM reduction of O.
//
// Restates model.py:229-253 (_attend) for forward_full (model.py:318-334) and
// forward_sparse (model.py:360-380), and the score path selection.py:78-135.
#include <cooperative_groups.h>

#include "common.cuh"

namespace cg = cooperative_groups;

namespace sd {
namespace tm_attn {

constexpr int TK = 64;   // keys per tile
constexpr int NCW = 8;   // math warps
constexpr int NT = (NCW + 1) * 32;
// Two shapes: V1 = one CTA per SM (10-slot ring, all 512 TMEM columns);
// V2 = two CTAs per SM (5-slot ring, 256 columns each) so one CTA's
// exchange / epilogue bubbles overlap the other's streaming.
constexpr float LOG2E = 1.4426950408889634f;
constexpr float LN2 = 0.6931471805599453f;

__device__ __forceinline__ unsigned smem_u32(const void* p) { return static_cast<unsigned>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
  asm volatile(
      "{\n.reg .pred p;\nWAIT_%=:\n"
      "mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
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
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;\n" : "=l"(p));
  return p;
}
__device__ __forceinline__ void cluster_arrive() { asm volatile("barrier.cluster.arrive.release.aligned;\n" ::: "memory"); }
__device__ __forceinline__ void cluster_wait() { asm volatile("barrier.cluster.wait.acquire.aligned;\n" ::: "memory"); }
__device__ __forceinline__ void math_bar() { asm volatile("bar.sync 1, %0;\n" ::"n"(NCW * 32) : "memory"); }

// ---- tensor memory ----
__device__ __forceinline__ void tmem_alloc(uint32_t* dst, int cols) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(dst)), "r"(cols));
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::);
}
__device__ __forceinline__ void tmem_dealloc(uint32_t taddr, int cols) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(taddr), "r"(cols));
}
__device__ __forceinline__ void tmem_st4(uint32_t taddr, const float (&v)[4]) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1, %2, %3, %4};\n" ::"r"(taddr),
               "r"(__float_as_uint(v[0])), "r"(__float_as_uint(v[1])), "r"(__float_as_uint(v[2])),
               "r"(__float_as_uint(v[3]))
               : "memory");
}
__device__ __forceinline__ void tmem_ld4(uint32_t taddr, float (&v)[4]) {
  uint32_t a, b, c, d;
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0, %1, %2, %3}, [%4];\n"
               : "=r"(a), "=r"(b), "=r"(c), "=r"(d)
               : "r"(taddr)
               : "memory");
  v[0] = __uint_as_float(a), v[1] = __uint_as_float(b), v[2] = __uint_as_float(c), v[3] = __uint_as_float(d);
}
__device__ __forceinline__ void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory"); }
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory"); }
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory"); }

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
__device__ __forceinline__ uint64_t gtime() {
  uint64_t t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
constexpr int kTraceCtas = 8192;
constexpr int kTraceSlots = 8;
__device__ uint64_t g_trace[kTraceCtas * kTraceSlots];

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
  int chunk;  // keys per CTA, multiple of TK, chunk/TK * MT * 4 <= HALF
  int nomath; // diagnostics: stream only (SD_ATTN_NOMATH=1)
  int trace;  // diagnostics: phase timestamps (SD_ATTN_TRACE=1)
};

struct Layout {
  int bar_off, tptr_off, ring_off, q_off, pos_off, slot_off, wm_off, wl_off, m_off, l_off, lse_off, total;
};
__host__ __device__ inline Layout make_layout(int D, int MT, int chunk, int NSLOT, int TCOLS) {
  const int RP = MT * 16;
  const int krow = D + 8;
  Layout L;
  int o = 0;
  L.bar_off = o;  o += 2 * NSLOT * 8;
  L.tptr_off = o; o += 16;
  o = (o + 127) & ~127;
  L.ring_off = o;
  {
    const int ring = NSLOT * TK * krow * 2;
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
  // >= 120 KB keeps occupancy at ONE CTA per SM: each CTA owns all 512 TMEM
  // columns, and two co-resident CTAs of one cluster would deadlock in alloc.
  L.total = (TCOLS == 512 && o < 120 * 1024) ? 120 * 1024 : o;
  return L;
}

template <int D, int MT, bool GM, int NSLOT, int TCOLS>
__global__ void __launch_bounds__(NT, TCOLS == 512 ? 1 : 2) attn_tm_kernel(const Params p) {
  constexpr int HALF = TCOLS / 2;  // TMEM columns per warp half (warps 0-3 / 4-7)
  constexpr int RP = MT * 16;
  constexpr int KROW = D + 8;
  constexpr int DCH = D / 8;
  constexpr int TILE = TK * KROW;
  constexpr int DH = D / 2;    // output columns per warp in phase 2
  constexpr int NTD = DH / 8;  // n8 tiles per warp in phase 2
  constexpr int TCPT = MT * 4;  // TMEM columns per tile per thread

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
  // diagnostics: per-CTA phase timestamps (SD_ATTN_TRACE=1, read with sd_attention_trace)
  const int cta_lin = (blockIdx.z * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x;
#define TRACE(k)                                                                                   \
  do {                                                                                             \
    if (p.trace && tid == 0 && cta_lin < kTraceCtas) g_trace[cta_lin * kTraceSlots + (k)] = gtime(); \
  } while (0)
  TRACE(0);

  extern __shared__ __align__(128) unsigned char smem[];
  const Layout L = make_layout(D, MT, p.chunk, NSLOT, TCOLS);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + L.bar_off);
  uint64_t* empty = full + NSLOT;
  uint32_t* tptr = reinterpret_cast<uint32_t*>(smem + L.tptr_off);
  __nv_bfloat16* ring = reinterpret_cast<__nv_bfloat16*>(smem + L.ring_off);
  __nv_bfloat16* Qs = reinterpret_cast<__nv_bfloat16*>(smem + L.q_off);
  int32_t* spos = reinterpret_cast<int32_t*>(smem + L.pos_off);
  int32_t* sslot = reinterpret_cast<int32_t*>(smem + L.slot_off);
  float* wm = reinterpret_cast<float*>(smem + L.wm_off);
  float* wl = reinterpret_cast<float*>(smem + L.wl_off);
  float* rowm = reinterpret_cast<float*>(smem + L.m_off);
  float* rowl = reinterpret_cast<float*>(smem + L.l_off);
  float* rowlse = reinterpret_cast<float*>(smem + L.lse_off);

  auto row_tok = [&](int r) { return GM ? (r & 7) : r / G; };
  auto row_g = [&](int r) { return GM ? (r >> 3) : r % G; };
  auto row_real = [&](int r) { return GM ? ((r & 7) < it.nq && (r >> 3) < G) : r < R; };

  // ---- setup ----
  if (warp == 0) tmem_alloc(tptr, TCOLS);
  if (tid < NSLOT) {
    mbar_init(full + tid, 32);
    mbar_init(empty + tid, NCW);
  }
  // key positions only (dense keys: arithmetic; critical keys: one load);
  // the producer resolves physical slots itself, one tile ahead
  for (int j = tid; j < ntiles * TK; j += NT) {
    const int gj = kb + j;
    spos[j] = gj < ke ? it.key_pos(p.crit, gj) : 0x7fffffff;
  }
  (void)sslot;
  for (int i = tid; i < RP * DCH; i += NT) {
    const int r = i / DCH, c = i - r * DCH;
    uint4 v = make_uint4(0, 0, 0, 0);
    if (row_real(r))
      v = *reinterpret_cast<const uint4*>(
          p.q + ((int64_t)(it.q_row0 + row_tok(r)) * p.q_heads + h * G + row_g(r)) * D + c * 8);
    *reinterpret_cast<uint4*>(Qs + r * KROW + c * 8) = v;
  }
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = *tptr;
  TRACE(1);

  const int kvh = p.kv.kv_heads;
  const __nv_bfloat16* Kg = static_cast<const __nv_bfloat16*>(p.kv.k) + (int64_t)p.layer * p.kv.layer_stride + h * D;
  const __nv_bfloat16* Vg = static_cast<const __nv_bfloat16*>(p.kv.v) + (int64_t)p.layer * p.kv.layer_stride + h * D;

  if (warp == NCW) {
    // ===================== producer =====================
    const uint64_t pol = policy_evict_first();  // every row is read exactly once
    const int last_valid = nk - 1;
    constexpr int KPI = 32 / DCH;  // key rows per warp instruction
    const int sub = lane / DCH, c = lane - sub * DCH;
    // physical slots of tile t's keys (lane, lane+32): block-table loads
    // issued one fill ahead so their latency overlaps the previous copies
    auto slots_of = [&](int t, int& s0, int& s1) {
      s0 = static_cast<int>(p.kv.slot_of(it.table_row, spos[min(t * TK + lane, last_valid)]));
      s1 = static_cast<int>(p.kv.slot_of(it.table_row, spos[min(t * TK + lane + 32, last_valid)]));
    };
    int slot0 = 0, slot1 = 0;
    if (ntiles > 0) slots_of(0, slot0, slot1);
    for (int f = 0; f < 2 * ntiles; ++f) {
      const int s = f % NSLOT;
      const int t = f < ntiles ? f : f - ntiles;
      const __nv_bfloat16* base = f < ntiles ? Kg : Vg;
      __nv_bfloat16* dst = ring + s * TILE;
      int n0s = 0, n1s = 0;
      if (f + 1 < 2 * ntiles) slots_of(f + 1 < ntiles ? f + 1 : f + 1 - ntiles, n0s, n1s);
      if (f >= NSLOT) mbar_wait(empty + s, ((f / NSLOT) - 1) & 1);
#pragma unroll 8
      for (int m = 0; m < TK / KPI; ++m) {
        const int kk = m * KPI + sub;
        const int sa = __shfl_sync(0xffffffffu, slot0, kk & 31);
        const int sb = __shfl_sync(0xffffffffu, slot1, kk & 31);
        cp_async16_pol(dst + kk * KROW + c * 8, base + (int64_t)(kk < 32 ? sa : sb) * (kvh * D) + c * 8, pol);
      }
      cp_async_mbar_arrive(full + s);
      slot0 = n0s;
      slot1 = n1s;
      if (f == ntiles - 1) cluster_arrive();  // K streamed: let the exchange proceed
    }
    if (ntiles == 0) cluster_arrive();
    cluster_wait();
    cluster_arrive();
    cluster_wait();
    cluster_arrive();
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
  const uint32_t tlane = tbase + ((uint32_t)(32 * (warp & 3)) << 16);
  const uint32_t tmine = tlane + (warp >> 2) * HALF;

  // ---- phase 1: S = Q K^T -> (max, sum), S -> TMEM ----
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
      float sacc[MT][4], sb[MT][4];
#pragma unroll
      for (int mt = 0; mt < MT; ++mt)
#pragma unroll
        for (int i = 0; i < 4; ++i) sacc[mt][i] = sb[mt][i] = 0.f;
      const __nv_bfloat16* Kt = ring + s * TILE;
#pragma unroll
      for (int ks = 0; ks < D / 16; ks += 2) {
        unsigned b0, b1, b2, b3;
        ldsm_x4(b0, b1, b2, b3, Kt + (n0 + (lane & 7)) * KROW + ks * 16 + (lane >> 3) * 8);
#pragma unroll
        for (int mt = 0; mt < MT; ++mt) {
          unsigned a0, a1, a2, a3;
          const __nv_bfloat16* qa = Qs + (mt * 16 + (lane & 7) + ((lane >> 3) & 1) * 8) * KROW + (lane >> 4) * 8;
          ldsm_x4(a0, a1, a2, a3, qa + ks * 16);
          mma_bf16(sacc[mt], a0, a1, a2, a3, b0, b1);
          ldsm_x4(a0, a1, a2, a3, qa + (ks + 1) * 16);
          mma_bf16(sb[mt], a0, a1, a2, a3, b2, b3);
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(empty + s);
      const bool fullt = tile_full(t);
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int jl = t * TK + n0 + 2 * t4 + e;
        const float bias = fullt ? 0.f : (p.n_planted ? planted_bias(p.planted, p.n_planted, p.bonus_log2, spos[jl]) : 0.f);
#pragma unroll
        for (int mt = 0; mt < MT; ++mt)
#pragma unroll
          for (int hh = 0; hh < 2; ++hh) {
            const int i = hh * 2 + e;
            const bool vis = fullt || visible(jl, mt * 16 + g4 + hh * 8);
            sacc[mt][i] = vis ? fmaf(sacc[mt][i] + sb[mt][i], p.scale_log2, bias) : -INFINITY;
          }
      }
#pragma unroll
      for (int mt = 0; mt < MT; ++mt) {
#pragma unroll
        for (int hh = 0; hh < 2; ++hh) {
          const float s0 = sacc[mt][hh * 2], s1 = sacc[mt][hh * 2 + 1];
          const float nm = fmaxf(pm[mt][hh], fmaxf(s0, s1));
          if (nm != -INFINITY) {
            pl[mt][hh] = pl[mt][hh] * ex2(pm[mt][hh] - nm) + ex2(s0 - nm) + ex2(s1 - nm);
            pm[mt][hh] = nm;
          }
        }
        tmem_st4(tmine + t * TCPT + mt * 4, sacc[mt]);
      }
    }
  }
  tmem_wait_st();
  TRACE(2);
  tc_fence_before();
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
  tc_fence_after();

  TRACE(3);
  // ---- phase 2: P = exp2(S - lse) from TMEM, scores, O = P V ----
  const int w4 = warp & 3;   // key pair: warps w4 and w4+4 own keys 8*w4.. and 8*w4+32..
  const int dh = warp >> 2;  // output-column half
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
    const int f = ntiles + t;
    const int s = f % NSLOT;
    if (p.nomath) {
      mbar_wait(full + s, (f / NSLOT) & 1);
      __syncwarp();
      if (lane == 0) mbar_arrive(empty + s);
      continue;
    }
    float P0[MT][4], P1[MT][4];  // keys of warp w4 / of warp w4+4
#pragma unroll
    for (int mt = 0; mt < MT; ++mt) {
      tmem_ld4(tlane + t * TCPT + mt * 4, P0[mt]);
      tmem_ld4(tlane + HALF + t * TCPT + mt * 4, P1[mt]);
    }
    tmem_wait_ld();
#pragma unroll
    for (int mt = 0; mt < MT; ++mt)
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const float l = lse_r[mt][i >> 1];
        P0[mt][i] = ex2(P0[mt][i] - l);
        P1[mt][i] = ex2(P1[mt][i] - l);
      }
    if (scores) {
#pragma unroll
      for (int half = 0; half < 2; ++half)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int jl = t * TK + 8 * (w4 + 4 * half) + 2 * t4 + e;
          const bool kvalid = kb + jl < ke;  // no early exit: the token-major path shuffles
          if constexpr (GM) {
            float v = 0.f;
#pragma unroll
            for (int mt = 0; mt < MT; ++mt) v += half ? P1[mt][e] + P1[mt][2 + e] : P0[mt][e] + P0[mt][2 + e];
            if (kvalid && g4 < it.nq && v != 0.f)
              atomicAdd(p.acc + (int64_t)(it.acc_row + g4 * it.acc_step) * p.acc_stride + spos[jl], v);
          } else {
            const int gl = min(G, 8);
#pragma unroll
            for (int mt = 0; mt < MT; ++mt) {
              float v0 = half ? P1[mt][e] : P0[mt][e];
              float v1 = half ? P1[mt][2 + e] : P0[mt][2 + e];
              if (G >= 16) v0 += v1;
              for (int o = 4; o < 4 * gl; o <<= 1) {
                v0 += __shfl_xor_sync(0xffffffffu, v0, o);
                v1 += __shfl_xor_sync(0xffffffffu, v1, o);
              }
              if (kvalid && (g4 % gl) == 0) {
                const int tok0 = (mt * 16 + g4) / G;
                if (v0 != 0.f && tok0 < it.nq)
                  atomicAdd(p.acc + (int64_t)(it.acc_row + tok0 * it.acc_step) * p.acc_stride + spos[jl], v0);
                if (G < 16) {
                  const int tok1 = (mt * 16 + g4 + 8) / G;
                  if (v1 != 0.f && tok1 < it.nq)
                    atomicAdd(p.acc + (int64_t)(it.acc_row + tok1 * it.acc_step) * p.acc_stride + spos[jl], v1);
                }
              }
            }
          }
        }
    }
    unsigned a[MT][4];
#pragma unroll
    for (int mt = 0; mt < MT; ++mt) {
      a[mt][0] = pack_bf16(P0[mt][0], P0[mt][1]);
      a[mt][1] = pack_bf16(P0[mt][2], P0[mt][3]);
      a[mt][2] = pack_bf16(P1[mt][0], P1[mt][1]);
      a[mt][3] = pack_bf16(P1[mt][2], P1[mt][3]);
    }
    mbar_wait(full + s, (f / NSLOT) & 1);
    const __nv_bfloat16* Vt = ring + s * TILE;
    // k16 rows: keys 8*w4 + 0..7 (lanes 0-7 / 16-23) and 8*w4 + 32..39 (lanes 8-15 / 24-31)
    const int vrow = 8 * w4 + (lane & 7) + ((lane >> 3) & 1) * 32;
#pragma unroll
    for (int nt = 0; nt < NTD; nt += 2) {
      unsigned b0, b1, b2, b3;
      ldsm_x4_t(b0, b1, b2, b3, Vt + vrow * KROW + dh * DH + nt * 8 + (lane >> 4) * 8);
#pragma unroll
      for (int mt = 0; mt < MT; ++mt) {
        mma_bf16(oacc[mt][nt], a[mt][0], a[mt][1], a[mt][2], a[mt][3], b0, b1);
        mma_bf16(oacc[mt][nt + 1], a[mt][0], a[mt][1], a[mt][2], a[mt][3], b2, b3);
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(empty + s);
  }

  TRACE(4);
  // ---- O partials: 4 key pairs -> smem (ring reused), cluster DSMEM reduce ----
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
  tc_fence_before();
  cluster_arrive();
  cluster_wait();
  for (int i = tid; i < ((RP - crank + C - 1) / C) * (D / 4); i += NCW * 32) {
    const int ri = i / (D / 4), c4 = i - ri * (D / 4);
    const int r = crank + ri * C;
    if (!row_real(r)) continue;
    float4 sum = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int c = 0; c < C; ++c) {
      const float4 v = *reinterpret_cast<const float4*>(cluster.map_shared_rank(Ob + r * D + c4 * 4, c));
      sum.x += v.x; sum.y += v.y; sum.z += v.z; sum.w += v.w;
    }
    __nv_bfloat162* dst = reinterpret_cast<__nv_bfloat162*>(
        p.out + ((int64_t)(it.q_row0 + row_tok(r)) * p.q_heads + h * G + row_g(r)) * D + c4 * 4);
    dst[0] = __floats2bfloat162_rn(sum.x, sum.y);
    dst[1] = __floats2bfloat162_rn(sum.z, sum.w);
  }
  if (p.lse_out != nullptr && crank == 0 && tid < RP && row_real(tid))
    p.lse_out[(int64_t)(it.q_row0 + row_tok(tid)) * p.q_heads + h * G + row_g(tid)] = rowlse[tid] * LN2;
  cluster_arrive();
  cluster_wait();
  tc_fence_after();
  if (warp == 0) tmem_dealloc(tbase, TCOLS);
  TRACE(5);
#undef TRACE
}

template <int D, int MT, bool GM, int NSLOT, int TCOLS>
int launch_one(const Params& prm, int C, int num_items, int kv_heads, cudaStream_t stream) {
  auto kern = attn_tm_kernel<D, MT, GM, NSLOT, TCOLS>;
  const int smem = make_layout(D, MT, prm.chunk, NSLOT, TCOLS).total;
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
    set_error(std::string("sd_attention (tmem) launch: ") + cudaGetErrorString(e));
    return (int)e;
  }
  return 0;
}

static int env_int(const char* name, int dflt) {
  const char* v = getenv(name);
  return v && *v ? atoi(v) : dflt;
}

}  // namespace tm_attn

// Cluster size: smallest C whose chunk fits the TMEM logit store, then the C
// (<= 16) that best fills whole waves of 148 single-CTA SMs.
static bool plan_tm(int max_keys, int num_items, int kv_heads, int MT, int tcols, int* C_out, int* chunk_out) {
  using namespace tm_attn;
  const int tiles = (max_keys + TK - 1) / TK;
  const int max_tiles = (tcols / 2) / (MT * 4);
  const int slots = 148 * (512 / tcols);
  const int c_min = (tiles + max_tiles - 1) / max_tiles;
  if (c_min > 16) return false;
  static const int force_c = env_int("SD_ATTN_C", 0);
  const int work = num_items * kv_heads;
  int best = c_min;
  double best_eff = -1.0;
  for (int c = c_min; c <= 16 && c <= tiles; ++c) {
    const int chunk_tiles = (tiles + c - 1) / c;
    const double ctas = (double)work * c;
    const double waves = ctas / (double)slots;
    // useful work per wave slot, penalising tiny chunks (fixed per-CTA cost ~1 tile)
    const double eff = (waves / (double)((long long)(waves + 0.999999))) * (chunk_tiles / (chunk_tiles + 1.0));
    if (eff > best_eff + 0.02) best_eff = eff, best = c;
  }
  if (force_c >= c_min && force_c <= 16) best = force_c;
  *C_out = best;
  *chunk_out = ((tiles + best - 1) / best) * TK;
  return true;
}

int launch_attn_tm(const void* q, void* out, float* lse, const sd_paged_kv* kvp, int layer, const int32_t* items,
                   int num_items, int max_keys, int max_nq, const int32_t* crit, float* acc, int64_t acc_stride,
                   const int32_t* planted, int n_planted, float bonus, int q_heads, float scale, cudaStream_t stream,
                   bool* handled) {
  using namespace tm_attn;
  const int D = kvp->head_dim;
  const int G = q_heads / kvp->kv_heads;
  *handled = false;
  if (kvp->dtype != SD_DTYPE_BF16 || !(D == 64 || D == 128)) return 0;
  const bool gm = max_nq >= 2 && max_nq <= 8 && G <= 8 && (G & (G - 1)) == 0 && G >= 2;
  const int rows = gm ? 8 * G : max_nq * G;
  if (rows > 80) return 0;
  const int MT = (rows + 15) / 16;
  static const int variant = env_int("SD_ATTN_TMV", 2);
  int tcols = variant == 1 ? 512 : 256;
  int C = 1, chunk = TK;
  if (!plan_tm(max_keys < 1 ? 1 : max_keys, num_items, kvp->kv_heads, MT, tcols, &C, &chunk)) {
    if (tcols == 512 || !plan_tm(max_keys < 1 ? 1 : max_keys, num_items, kvp->kv_heads, MT, 512, &C, &chunk)) return 0;
    tcols = 512;  // long context: fall back to the one-CTA-per-SM shape
  }
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
  static const int trace = env_int("SD_ATTN_TRACE", 0);
  prm.trace = trace;
  *handled = true;
#define SD_TM_CASE(DD, M)                                                                             \
  if (D == DD && MT == M) {                                                                           \
    if (tcols == 512) {                                                                               \
      if (gm) return launch_one<DD, M, true, 10, 512>(prm, C, num_items, kvp->kv_heads, stream);      \
      return launch_one<DD, M, false, 10, 512>(prm, C, num_items, kvp->kv_heads, stream);             \
    }                                                                                                 \
    if (gm) return launch_one<DD, M, true, 5, 256>(prm, C, num_items, kvp->kv_heads, stream);         \
    return launch_one<DD, M, false, 5, 256>(prm, C, num_items, kvp->kv_heads, stream);                \
  }
  SD_TM_CASE(128, 1) SD_TM_CASE(128, 2) SD_TM_CASE(128, 3) SD_TM_CASE(128, 4) SD_TM_CASE(128, 5)
  SD_TM_CASE(64, 1) SD_TM_CASE(64, 2) SD_TM_CASE(64, 3) SD_TM_CASE(64, 4) SD_TM_CASE(64, 5)
#undef SD_TM_CASE
  *handled = false;
  return 0;
}

}  // namespace sd

// Diagnostics: copy the per-CTA phase timestamps of the last traced launch
// (SD_ATTN_TRACE=1) to host memory: [ctas][8] uint64 globaltimer ns.
extern "C" int sd_attention_trace(uint64_t* host_dst, int32_t ctas) {
  if (ctas > sd::tm_attn::kTraceCtas) ctas = sd::tm_attn::kTraceCtas;
  cudaError_t e = cudaMemcpyFromSymbol(host_dst, sd::tm_attn::g_trace,
                                       sizeof(uint64_t) * sd::tm_attn::kTraceSlots * ctas);
  return e == cudaSuccess ? 0 : (int)e;
}
