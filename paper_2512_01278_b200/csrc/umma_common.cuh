// Shared device helpers of the tcgen05 attention kernels (attn_umma.cu, attn_umma_pk.cu):
// mbarriers, cp.async, TMEM, UMMA descriptors, launch parameters and the smem layout.
#pragma once
#include <cooperative_groups.h>
#include <cuda.h>

#include "common.cuh"

namespace cg = cooperative_groups;

namespace sd {
namespace umma_attn {

constexpr int TK = 128;                 // keys per tile = UMMA M
constexpr int D = 128;                  // head dim (two 64-element swizzle atoms)
constexpr int NSW = 4;                  // softmax warps
constexpr int WPROD = 4, WMMA = 5;
constexpr int NT = 6 * 32;
constexpr int TILE_BYTES = TK * D * 2;  // 32 KB
constexpr float LOG2E = 1.4426950408889634f;
constexpr float LN2 = 0.6931471805599453f;

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
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
__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src, uint64_t policy) {
  asm volatile("cp.async.cg.shared.global.L2::cache_hint [%0], [%1], 16, %2;\n" ::"r"(dst), "l"(src), "l"(policy)
               : "memory");
}
__device__ __forceinline__ void cp_async_mbar_arrive(uint64_t* bar) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_arrive_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
// TMA: one 16-key x 64-element box of a K or V page into the SWIZZLE_128B tile layout
__device__ __forceinline__ void tma_box(uint32_t dst, const CUtensorMap* map, int c0, int c1, int c2, uint64_t* bar,
                                        uint64_t pol) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%2, %3, %4}], [%5], %6;\n" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar)), "l"(pol)
      : "memory");
}
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;\n" : "=l"(p));
  return p;
}
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory"); }
__device__ __forceinline__ void cluster_arrive() { asm volatile("barrier.cluster.arrive.release.aligned;\n" ::: "memory"); }
__device__ __forceinline__ void cluster_wait() { asm volatile("barrier.cluster.wait.acquire.aligned;\n" ::: "memory"); }
__device__ __forceinline__ void sw_bar() { asm volatile("bar.sync 1, %0;\n" ::"n"(NSW * 32) : "memory"); }
__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;\n" : "=f"(y) : "f"(x));
  return y;
}
// PillarAttn score accumulation in fixed point: v = round(p * 2^shift) added with an
// integer reduction, so the sum over heads, CTAs and layers is independent of the
// order the atomics land in (bitwise reproducible importance; see spardec_b200.h)
__device__ __forceinline__ void red_add_fx(unsigned long long* p, float v, float scale) {
  const unsigned long long u = __float2ull_rn(v * scale);
  if (u != 0ull) asm volatile("red.global.add.u64 [%0], %1;\n" ::"l"(p), "l"(u) : "memory");
}

// ---- tensor memory / UMMA ----
__device__ __forceinline__ void tmem_alloc(uint32_t* dst, int cols) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(dst)), "r"(cols));
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::);
}
__device__ __forceinline__ void tmem_dealloc(uint32_t taddr, int cols) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(taddr), "r"(cols));
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory"); }
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory"); }

// 16 consecutive fp32 columns of this thread's TMEM lane
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float* v) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];\n"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr)
      : "memory");
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}
__device__ __forceinline__ void tmem_ld8(uint32_t taddr, float* v) {
  uint32_t r[8];
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];\n"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
               : "r"(taddr)
               : "memory");
#pragma unroll
  for (int i = 0; i < 8; ++i) v[i] = __uint_as_float(r[i]);
}
// N (a multiple of 8) consecutive fp32 columns, issued back to back; caller waits
template <int N>
__device__ __forceinline__ void tmem_ld_cols(uint32_t taddr, float* v) {
  static_assert(N % 8 == 0, "TMEM column group must be a multiple of 8");
#pragma unroll
  for (int c = 0; c + 16 <= N; c += 16) tmem_ld16(taddr + c, v + c);
  if constexpr (N % 16 == 8) tmem_ld8(taddr + N - 8, v + N - 8);
}
template <int NR>
__device__ __forceinline__ void tmem_ld_row(uint32_t taddr, float (&v)[NR]) {
  tmem_ld_cols<NR>(taddr, v);
  tmem_wait_ld();
}

// SM100 shared-memory matrix descriptor (start, LBO, SBO in 16-byte units,
// version 1, layout type in bits 61-63: 0 = no swizzle, 2 = 128-byte swizzle)
__device__ __forceinline__ uint64_t smem_desc(uint32_t addr, uint32_t lbo, uint32_t sbo, uint32_t layout) {
  return (uint64_t)((addr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | (1ull << 46) | ((uint64_t)layout << 61);
}
// kind::f16 instruction descriptor: bf16 x bf16 -> f32, M = 128, N = n
__device__ __forceinline__ uint32_t idesc_bf16(int n, bool a_mn_major, bool b_mn_major) {
  return (1u << 4)                        // D format f32
         | (1u << 7) | (1u << 10)         // A, B format bf16
         | ((a_mn_major ? 1u : 0u) << 15) | ((b_mn_major ? 1u : 0u) << 16) |
         ((uint32_t)(n >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
}
__device__ __forceinline__ void umma(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t accum) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
      "l"(a), "l"(b), "r"(idesc), "r"(accum));
}
__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(smem_u32(bar))
               : "memory");
}

constexpr int kTraceCtas = 16384;
constexpr int kTraceSlots = 12;
__device__ __forceinline__ uint64_t gtime() {
  uint64_t t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

struct Params {
  CUtensorMap tmk;  // dense items: the layer's K / V pool as [slots][kv heads][128] bf16,
  CUtensorMap tmv;  // 16-slot x 1-head x 64-element boxes, SWIZZLE_128B (valid when tma)
  int tma;
  uint64_t* trace;  // diagnostics: [kTraceCtas][kTraceSlots] per-CTA phase timestamps, or null
  const __nv_bfloat16* q;
  __nv_bfloat16* out;
  float* lse_out;
  PagedKv kv;
  int layer;
  const int32_t* items;
  const int32_t* crit;
  unsigned long long* acc;  // fixed-point score accumulators (2^acc_shift per unit)
  int64_t acc_stride;
  float acc_scale;           // 2^acc_shift
  const int32_t* planted;
  int n_planted;
  float bonus_log2;
  int q_heads;
  float scale_log2;
  int chunk;  // keys per CTA, multiple of TK
  int dense;  // 1: items have no critical list and pages >= 16 tokens (page ids staged, not slots)
};

// (m, l) softmax-statistics merge
__device__ __forceinline__ void stat_merge(float& m, float& l, float om, float ol) {
  const float nm = fmaxf(m, om);
  l = (nm == -INFINITY) ? 0.f : l * ex2(m - nm) + ol * ex2(om - nm);
  m = nm;
}
// Transpose-reduce N (power of two <= 32) per-row statistics over the warp's 32 keys:
// halving rounds exchange half of the rows each time (N - 1 shuffles per value instead
// of 5N), leaving lane L with the full reduction of row L % N in m[0], l[0].
template <int N>
__device__ __forceinline__ void warp_rows_reduce(float* m, float* l, int lane) {
#pragma unroll
  for (int o = N / 2; o >= 1; o >>= 1) {
    const bool hi = (lane & o) != 0;
#pragma unroll
    for (int i = 0; i < o; ++i) {
      const float sm = hi ? m[i] : m[i + o], sl = hi ? l[i] : l[i + o];
      float km = hi ? m[i + o] : m[i], kl = hi ? l[i + o] : l[i];
      const float rm = __shfl_xor_sync(0xffffffffu, sm, o), rl = __shfl_xor_sync(0xffffffffu, sl, o);
      stat_merge(km, kl, rm, rl);
      m[i] = km, l[i] = kl;
    }
  }
#pragma unroll
  for (int o = N; o < 32; o <<= 1) {
    const float rm = __shfl_xor_sync(0xffffffffu, m[0], o), rl = __shfl_xor_sync(0xffffffffu, l[0], o);
    stat_merge(m[0], l[0], rm, rl);
  }
}

struct Layout {
  int ring, q, pbuf, pos, slot, bar, wm, wl, xm, xl, rowlse, tptr, total;
};
__host__ __device__ constexpr int align_up(int x, int a) { return (x + a - 1) / a * a; }
// ct = key tiles of this launch's chunk.  Gathered (critical-list) items stage a position
// and a physical slot per key; dense items (dense = 1: no critical list, pages of >= 16
// tokens) only the chunk's block-table entries, one per page.
__host__ __device__ inline Layout make_layout(int NR, int NSLOT, int S, int ct, int dense = 0) {
  Layout L{};
  int o = 0;
  L.ring = o;  o += NSLOT * TILE_BYTES;
  L.q = o;     o += 2 * NR * 128;        // [dhalf][NR][128 B], SWIZZLE_128B
  L.pbuf = o;  o += 2 * NR * TK * 2;     // 2 x P^T [128 keys][NR] bf16, MN-major, no swizzle
  L.pos = o;   o += dense ? (ct * TK / 16 + 2) * 4 : ct * TK * 4;
  L.slot = o;  o += dense ? 0 : ct * TK * 4;
  o = align_up(o, 8);
  L.bar = o;   o += (2 * NSLOT + 2 * S + 6) * 8;
  L.wm = o;    o += NSW * NR * 4;
  L.wl = o;    o += NSW * NR * 4;
  L.xm = o;    o += 16 * NR * 4;          // [source CTA][row] pushed by every cluster peer
  L.xl = o;    o += 16 * NR * 4;
  L.rowlse = o; o += NR * 4;
  L.tptr = o;  o += 16;
  L.total = align_up(o, 128) + 1024;  // + slack to 1024-align the dynamic base
  return L;
}

}  // namespace umma_attn
}  // namespace sd
