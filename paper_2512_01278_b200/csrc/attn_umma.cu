// tcgen05 attention dispatch for sm_100a: the head-packed K1 draft kernel (this file), the
// K2 verify kernel (attn_umma.cuh, instantiated per GQA group in attn_umma_g4/g8.cu) and
// the launch planner that picks the cluster split.
#include "attn_umma.cuh"

#include <map>
#include <mutex>
#include <algorithm>
#include <tuple>

#include <cuda.h>

namespace sd {
namespace umma_attn {

// Fill order of the head-packed kernel's producer ring (each fill = one 32 KB K or V tile):
//   K[0..nt), V[nt-TR..nt) over the TMEM-resident tiles, then (K[j], V[j]) j < nt-TR
__device__ __forceinline__ void fill_tile_hp(int f, int nt, int TR, int& t, bool& isv) {
  if (f < nt) {
    t = f, isv = false;
  } else if (f < nt + TR) {
    t = nt - TR + (f - nt), isv = true;
  } else {
    const int g = f - nt - TR;
    t = g >> 1, isv = g & 1;
  }
}

// ---------------------------------------------------------------------------------------
// Head-packed draft kernel (K1, one query token per item): a CTA covers HPC kv heads of one
// item, and a 128-row UMMA tile is KPT = 128 / HPC keys x HPC heads (head-major rows), so
//   S^T[(head, key)][HPC*G] = K_rows . Q^T      (only the row's own head block is used)
//   O^T[d][HPC*G]         += V_rows^T . P^T    (P^T is block-diagonal: exact per head)
// Every statistic of a (head, q head) row lives inside one warp (KPT = 32 or 16 keys of the
// tile per head), so there is no CTA exchange; the setup cost is paid once per HPC heads
// and every fill moves 32 KB however small the critical set is.
template <int N>
__device__ __forceinline__ void tmem_ld_n(uint32_t taddr, float* v) {
  if constexpr (N == 4) {
    uint32_t r0, r1, r2, r3;
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];\n"
                 : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3) : "r"(taddr) : "memory");
    v[0] = __uint_as_float(r0), v[1] = __uint_as_float(r1), v[2] = __uint_as_float(r2), v[3] = __uint_as_float(r3);
  } else if constexpr (N == 8) {
    uint32_t r[8];
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];\n"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
                 : "r"(taddr) : "memory");
#pragma unroll
    for (int i = 0; i < 8; ++i) v[i] = __uint_as_float(r[i]);
  } else {
    static_assert(N % 16 == 0, "tcgen05.ld width");
#pragma unroll
    for (int c = 0; c < N; c += 16) tmem_ld16(taddr + c, v + c);
  }
}

// shared-memory layout of the head-packed kernel: no cross-warp statistics arrays
__host__ __device__ inline Layout make_hp_layout(int NR, int NSLOT, int TMAX, int ct) {
  Layout L{};
  int o = 0;
  L.ring = o;  o += NSLOT * TILE_BYTES;
  L.q = o;     o += 2 * NR * 128;
  L.pbuf = o;  o += 2 * NR * TK * 2;
  L.pos = o;   o += ct * TK * 4;
  L.slot = o;  o += ct * TK * 4;
  o = align_up(o, 8);
  L.bar = o;   o += (2 * NSLOT + 2 * TMAX + 5) * 8;
  L.tptr = o;  o += 16;
  L.wm = L.wl = L.xm = L.xl = L.rowlse = 0;
  L.total = align_up(o, 128) + 1024;
  return L;
}

// head-packed kernel warp layout: softmax warps 0-3, HP_NPROD producer warps, the MMA warp
constexpr int HP_NPROD = 4;
constexpr int HP_WPROD = NSW, HP_WMMA = NSW + HP_NPROD;
constexpr int HP_NT = (NSW + HP_NPROD + 1) * 32;

template <int G, int HPC, int NSLOT, int TCOLS>
__device__ __forceinline__ void draft_body(const Params& p, const int hgroup, const int item_idx) {
  constexpr int NQ = HPC * G;                       // q heads of the CTA
  constexpr int NR = NQ < 16 ? 16 : NQ;             // UMMA N
  constexpr int KPT = TK / HPC;                     // keys per tile
  constexpr int TMAX = (TCOLS - NR) / NR;
  constexpr int OCOL = TMAX * NR;
  constexpr int WH = KPT >= 32 ? 1 : 32 / KPT;      // heads per warp (rows of a warp)
  static_assert(KPT == 16 || KPT == 32, "head packing: 4 or 8 heads per CTA");

  const int h0 = hgroup * HPC;
  const Item it = load_item(p.items, item_idx);
  const int nk = it.num_keys();
  const int nt = (nk + KPT - 1) / KPT;
  const int TR = min(nt, TMAX);
  const int nfill = 3 * nt - TR;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int cta_lin = blockIdx.y * gridDim.x + blockIdx.x;
#define HTRACE(k, val)                                                                                  \
  do {                                                                                                  \
    if (p.trace && cta_lin < kTraceCtas) p.trace[cta_lin * kTraceSlots + (k)] = (val);                  \
  } while (0)
  if (tid == 0) {
    uint32_t smid;
    asm volatile("mov.u32 %0, %smid;" : "=r"(smid));
    HTRACE(0, gtime());
    HTRACE(9, (uint64_t)smid | ((uint64_t)nt << 32));
  }

  extern __shared__ unsigned char smem_raw[];
  unsigned char* smem = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const Layout L = make_hp_layout(NR, NSLOT, TMAX, (nt * KPT + TK - 1) / TK);
  unsigned char* ring = smem + L.ring;
  unsigned char* qs = smem + L.q;
  unsigned char* pbuf = smem + L.pbuf;
  int32_t* spos = reinterpret_cast<int32_t*>(smem + L.pos);
  int32_t* sslot = reinterpret_cast<int32_t*>(smem + L.slot);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + L.bar);
  uint64_t* empty = full + NSLOT;
  uint64_t* sfull = empty + NSLOT;
  uint64_t* sfree = sfull + TMAX;
  uint64_t* pready = sfree + TMAX;
  uint64_t* pfree = pready + 2;
  uint64_t* obar = pfree + 2;
  uint32_t* tptr = reinterpret_cast<uint32_t*>(smem + L.tptr);

  if (warp == HP_WMMA) tmem_alloc(tptr, TCOLS);
  if (tid == 0) {
    for (int i = 0; i < NSLOT; ++i) mbar_init(full + i, 32 * HP_NPROD), mbar_init(empty + i, 1);
    for (int i = 0; i < TMAX; ++i) mbar_init(sfull + i, 1), mbar_init(sfree + i, NSW);
    mbar_init(pready + 0, NSW), mbar_init(pready + 1, NSW);
    mbar_init(pfree + 0, 1), mbar_init(pfree + 1, 1);
    mbar_init(obar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  {
    const int nkeys = nt * KPT;
    const int32_t* trow = p.kv.table + (int64_t)it.table_row * p.kv.table_stride;
    const int pmask = (1 << p.kv.page_shift) - 1;
    for (int j0 = 0; j0 < nkeys; j0 += 8 * HP_NT) {
      int pos[8], pg[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) pos[k] = it.key_pos(p.crit, min(j0 + k * HP_NT + tid, nk - 1));
#pragma unroll
      for (int k = 0; k < 8; ++k) pg[k] = __ldg(trow + (pos[k] >> p.kv.page_shift));
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const int j = j0 + k * HP_NT + tid;
        if (j < nkeys) {
          spos[j] = j < nk ? pos[k] : -1;
          sslot[j] = (pg[k] << p.kv.page_shift) | (pos[k] & pmask);
        }
      }
    }
  }
  // Q: the CTA's NQ q heads are contiguous in the row (heads h0.. x group)
  for (int i = tid; i < NR * 16; i += HP_NT) {
    const int r = i >> 4, c = i & 15;
    uint4 v = make_uint4(0, 0, 0, 0);
    if (r < NQ) v = *reinterpret_cast<const uint4*>(p.q + ((int64_t)it.q_row0 * p.q_heads + h0 * G + r) * D + c * 8);
    *reinterpret_cast<uint4*>(qs + (c >> 3) * (NR * 128) + r * 128 + (((c & 7) ^ (r & 7)) << 4)) = v;
  }
  // P^T buffers: off-diagonal blocks stay zero for the whole launch
  for (int i = tid; i < 2 * NR * TK * 2 / 16; i += HP_NT) reinterpret_cast<uint4*>(pbuf)[i] = make_uint4(0, 0, 0, 0);
  fence_proxy_async();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = *tptr;
  if (tid == 0) HTRACE(1, gtime());

  const int64_t row_stride = (int64_t)p.kv.kv_heads * D;
  const __nv_bfloat16* Kg = static_cast<const __nv_bfloat16*>(p.kv.k) + (int64_t)p.layer * p.kv.layer_stride + h0 * D;
  const __nv_bfloat16* Vg = static_cast<const __nv_bfloat16*>(p.kv.v) + (int64_t)p.layer * p.kv.layer_stride + h0 * D;

  if (warp >= HP_WPROD && warp < HP_WPROD + HP_NPROD) {
    // producers: warp pw copies rows [pw * 128 / HP_NPROD, ...) of every 32 KB fill (one head's keys)
    const int pw = warp - HP_WPROD;
    const uint64_t pol = policy_evict_first();
    const int sub = lane >> 4, c = lane & 15;
    const uint32_t ring_u = smem_u32(ring);
    constexpr int KK = TK / 2 / HP_NPROD;  // row pairs per warp
    for (int f = 0; f < nfill; ++f) {
      const int s = f % NSLOT;
      int t;
      bool isv;
      fill_tile_hp(f, nt, TR, t, isv);
      const __nv_bfloat16* base = (isv ? Vg : Kg) + c * 8;
      const int sl = sslot[t * KPT + (lane % KPT)];
      if (f >= NSLOT) mbar_wait(empty + s, ((f / NSLOT) - 1) & 1);
      const uint32_t dst0 = ring_u + s * TILE_BYTES + (c >> 3) * (TK * 128);
#pragma unroll
      for (int k2 = 0; k2 < KK; ++k2) {
        const int kk = pw * KK + k2;
        const int i = 2 * kk + sub;            // tile row = head-major (hh, key)
        const int hh = (2 * kk) / KPT;         // same for both rows of the instruction
        const int slot = __shfl_sync(0xffffffffu, sl, ((2 * kk) % KPT) + sub);
        cp_async16(dst0 + i * 128 + (((c & 7) ^ (i & 7)) << 4), base + (int64_t)slot * row_stride + hh * D, pol);
      }
      cp_async_mbar_arrive(full + s);
    }
    if (pw == 0 && lane == 0) HTRACE(7, gtime());
    return;
  }

  if (warp == HP_WMMA) {
    const uint32_t ring_u = smem_u32(ring), q_u = smem_u32(qs), p_u = smem_u32(pbuf);
    const uint32_t id_qk = idesc_bf16(NR, false, false);
    const uint32_t id_pv = idesc_bf16(NR, true, true);
    const bool leader = lane == 0;
    int f = 0;
    auto qk = [&](int u, int s) {
      mbar_wait(full + s, (f / NSLOT) & 1);
      if (u >= TMAX) mbar_wait(sfree + u % TMAX, ((u / TMAX) - 1) & 1);
      fence_proxy_async();
      tc_fence_after();
      if (leader) {
        const uint32_t a0 = ring_u + s * TILE_BYTES;
#pragma unroll
        for (int ks = 0; ks < D / 16; ++ks) {
          const uint32_t off = (ks & 3) << 5;
          const uint64_t a = smem_desc(a0 + (ks >> 2) * (TK * 128) + off, 16, 1024, 2);
          const uint64_t b = smem_desc(q_u + (ks >> 2) * (NR * 128) + off, 16, 1024, 2);
          umma(tbase + (u % TMAX) * NR, a, b, id_qk, ks > 0);
        }
        umma_commit(empty + s);
        umma_commit(sfull + u % TMAX);
      }
      __syncwarp();
      ++f;
    };
    for (int t = 0; t < nt; ++t) qk(t, f % NSLOT);
    for (int i2 = 0; i2 < nt; ++i2) {
      if (i2 >= TR) qk(nt + (i2 - TR), f % NSLOT);
      const int s = f % NSLOT;
      mbar_wait(full + s, (f / NSLOT) & 1);
      mbar_wait(pready + (i2 & 1), (i2 >> 1) & 1);
      fence_proxy_async();
      tc_fence_after();
      if (leader) {
        const uint32_t a0 = ring_u + s * TILE_BYTES;
        const uint32_t b0 = p_u + (i2 & 1) * (NR * TK * 2);
#pragma unroll
        for (int ks = 0; ks < TK / 16; ++ks) {
          const uint64_t a = smem_desc(a0 + ks * 16 * 128, TK * 128, 1024, 2);
          const uint64_t b = smem_desc(b0 + ks * 2 * 128, 128, TK * 16, 0);
          umma(tbase + OCOL, a, b, id_pv, (i2 > 0 || ks > 0) ? 1u : 0u);
        }
        umma_commit(empty + s);
        umma_commit(pfree + (i2 & 1));
        if (i2 == nt - 1) umma_commit(obar);
      }
      __syncwarp();
      ++f;
    }
    asm volatile("bar.sync 2, %0;\n" ::"n"((NSW + 1) * 32) : "memory");
    tc_fence_after();
    tmem_dealloc(tbase, TCOLS);
    return;
  }

  // ===================== softmax warps: thread = (head, key) row of the tile =====================
  const int row = warp * 32 + lane;
  const int hh = row / KPT, k = row % KPT;
  const int hsel = WH > 1 ? (lane / KPT) : 0;            // which of the warp's heads
  const int col0 = (warp * 32 / KPT) * G;                // first S column the warp reads
  const uint32_t tl = tbase + ((uint32_t)(warp * 32) << 16);
  float m[G], l[G];
#pragma unroll
  for (int g = 0; g < G; ++g) m[g] = -INFINITY, l[g] = 0.f;

  auto load_s = [&](int u, float (&v)[G]) {
    float w[WH * G];
    tmem_ld_n<WH * G>(tl + (u % TMAX) * NR + col0, w);
    tmem_wait_ld();
#pragma unroll
    for (int g = 0; g < G; ++g) v[g] = WH > 1 && hsel ? w[G + g] : w[g];
  };
  auto key_info = [&](int t, int& pos, float& bias, bool& vis) {
    const int j = t * KPT + k;
    pos = spos[j];
    vis = pos >= 0 && (j < it.crit_len || pos <= it.qpos0);
    bias = (vis && p.n_planted) ? planted_bias(p.planted, p.n_planted, p.bonus_log2, pos) : 0.f;
  };
  auto release = [&](int u) {
    tc_fence_before();
    __syncwarp();
    if (lane == 0) mbar_arrive(sfree + u % TMAX);
  };

  for (int t = 0; t < nt; ++t) {
    int pos;
    float bias;
    bool vis;
    key_info(t, pos, bias, vis);
    mbar_wait(sfull + t % TMAX, (t / TMAX) & 1);
    tc_fence_after();
    float v[G];
    load_s(t, v);
    if (t < nt - TR) release(t);
    if (vis) {
#pragma unroll
      for (int g = 0; g < G; ++g) {
        const float s2 = fmaf(v[g], p.scale_log2, bias);
        const float nm = fmaxf(m[g], s2);
        l[g] = l[g] * ex2(m[g] - nm) + ex2(s2 - nm);
        m[g] = nm;
      }
    }
  }
  // statistics of each (head, q head) row: reduce over the KPT lanes of this head
  float lse[G];
#pragma unroll
  for (int g = 0; g < G; ++g) {
#pragma unroll
    for (int o = KPT / 2; o >= 1; o >>= 1) {
      const float om = __shfl_xor_sync(0xffffffffu, m[g], o), ol = __shfl_xor_sync(0xffffffffu, l[g], o);
      stat_merge(m[g], l[g], om, ol);
    }
    lse[g] = m[g] + log2f(l[g]);
  }
  if (tid == 0) {
    HTRACE(2, gtime());
    HTRACE(3, gtime());
  }

  const bool scores = p.acc != nullptr && it.acc_row >= 0;
  for (int i2 = 0; i2 < nt; ++i2) {
    const int t = i2 < TR ? nt - TR + i2 : i2 - TR;
    const int u = i2 < TR ? t : nt + t;
    int pos;
    float bias;
    bool vis;
    key_info(t, pos, bias, vis);
    mbar_wait(sfull + u % TMAX, (u / TMAX) & 1);
    tc_fence_after();
    float v[G];
    load_s(u, v);
    release(u);
    float sum = 0.f;
#pragma unroll
    for (int g = 0; g < G; ++g) {
      v[g] = vis ? ex2(fmaf(v[g], p.scale_log2, bias) - lse[g]) : 0.f;
      sum += v[g];
    }
    if (scores && sum != 0.f) red_add_fx(p.acc + (int64_t)it.acc_row * p.acc_stride + pos, sum, p.acc_scale);
    if (i2 >= 2) mbar_wait(pfree + (i2 & 1), ((i2 >> 1) - 1) & 1);
    // P^T row `row`: this head's G columns (the rest of the row stays zero)
    unsigned char* pb = pbuf + (i2 & 1) * (NR * TK * 2) + row * 16 + ((hh * G) >> 3) * (TK * 16);
    if constexpr (G == 8) {
      uint4 w;
      __nv_bfloat162 b0 = __floats2bfloat162_rn(v[0], v[1]), b1 = __floats2bfloat162_rn(v[2], v[3]);
      __nv_bfloat162 b2 = __floats2bfloat162_rn(v[4], v[5]), b3 = __floats2bfloat162_rn(v[6], v[7]);
      w.x = *reinterpret_cast<uint32_t*>(&b0), w.y = *reinterpret_cast<uint32_t*>(&b1);
      w.z = *reinterpret_cast<uint32_t*>(&b2), w.w = *reinterpret_cast<uint32_t*>(&b3);
      *reinterpret_cast<uint4*>(pb) = w;
    } else {
      static_assert(G == 4, "group size 4 or 8");
      uint2 w;
      __nv_bfloat162 b0 = __floats2bfloat162_rn(v[0], v[1]), b1 = __floats2bfloat162_rn(v[2], v[3]);
      w.x = *reinterpret_cast<uint32_t*>(&b0), w.y = *reinterpret_cast<uint32_t*>(&b1);
      *reinterpret_cast<uint2*>(pb + ((hh * G) & 7) * 2) = w;
    }
    fence_proxy_async();
    __syncwarp();
    if (lane == 0) mbar_arrive(pready + (i2 & 1));
  }

  float o[NR];
  if (tid == 0) HTRACE(4, gtime());
  if (nt > 0) {
    mbar_wait(obar, 0);
    tc_fence_after();
    if (tid == 0) HTRACE(5, gtime());
    tmem_ld_row<NR>(tl + OCOL, o);
  } else {
#pragma unroll
    for (int r = 0; r < NR; ++r) o[r] = 0.f;
  }
  tc_fence_before();
  asm volatile("bar.arrive 2, %0;\n" ::"n"((NSW + 1) * 32) : "memory");
#pragma unroll
  for (int r = 0; r < NQ; ++r)
    p.out[((int64_t)it.q_row0 * p.q_heads + h0 * G + r) * D + row] = __float2bfloat16_rn(o[r]);
  if (p.lse_out != nullptr && k == 0) {
#pragma unroll
    for (int g = 0; g < G; ++g) p.lse_out[(int64_t)it.q_row0 * p.q_heads + (h0 + hh) * G + g] = lse[g] * LN2;
  }
  if (tid == 0) HTRACE(6, gtime());
#undef HTRACE
}

template <int G, int HPC, int NSLOT, int TCOLS>
__global__ void __launch_bounds__(HP_NT, TCOLS == 512 ? 1 : 2) attn_umma_hp_kernel(const __grid_constant__ Params p) {
  draft_body<G, HPC, NSLOT, TCOLS>(p, blockIdx.x, blockIdx.y);
}

template <int G, int HPC, int NSLOT, int TCOLS>
int launch_hp(const Params& prm, int num_items, int kv_heads, int ct, cudaStream_t stream) {
  constexpr int NQ = HPC * G, NR = NQ < 16 ? 16 : NQ, TMAX = (TCOLS - NR) / NR;
  auto kern = attn_umma_hp_kernel<G, HPC, NSLOT, TCOLS>;
  const int smem = make_hp_layout(NR, NSLOT, TMAX, ct).total;
  static int configured = 0;
  if (smem > configured) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, 100);  // as K2: no reconfig
    configured = smem;
  }
  kern<<<dim3(kv_heads / HPC, num_items), HP_NT, smem, stream>>>(prm);
  count_launch();
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_error(std::string("sd_attention (umma, head-packed) launch: ") + cudaGetErrorString(e));
    return (int)e;
  }
  return 0;
}

static uint64_t* g_trace_buf = nullptr;  // SD_ATTN_TRACE=1: per-CTA phase timestamps

static int env_int(const char* name, int dflt) {
  const char* v = getenv(name);
  return v && *v ? atoi(v) : dflt;
}

// Key tiles of one CTA's chunk that fit the shared-memory budget (positions + slots staged per key).
static int chunk_cap_tiles(int NR, int nslot, int S, int budget, int dense) {
  int ct = 1;
  while (ct < 512 && make_layout(NR, nslot, S, ct + 1, dense).total <= budget) ++ct;
  return make_layout(NR, nslot, S, ct, dense).total <= budget ? ct : 0;
}

}  // namespace umma_attn

// Cluster size C (<= 16) and chunk for one launch: minimise (waves of CTA slots) x
// (32 KB fills per CTA + a fixed per-CTA cost in fills, fitted to traced C sweeps).  Chunks
// longer than the S TMEM-resident tiles re-read the evicted tiles' K in phase 2
// (fills = 3*ct - S instead of 2*ct).
template <typename SlotsFn>
static bool plan_umma(int max_keys, int num_items, int kv_heads, int S, int cap, SlotsFn slots_of, int* C_out,
                      int* chunk_out, int dense) {
  using namespace umma_attn;
  const int tiles = (max_keys + TK - 1) / TK;
  static const int force_c = env_int("SD_ATTN_C", 0);
  // fixed per-CTA cost in fills: ~7 for dense verify chunks (traced C sweeps); re-reading an
  // evicted tile of a gathered (critical-list) chunk costs a second gather, so gathered
  // launches weight the per-CTA cost less and avoid re-reads
  static const double ovh_dense = env_int("SD_UMMA_OVH10", 70) / 10.0;
  const double ovh = dense ? ovh_dense : 2.0;
  const long long work = (long long)num_items * kv_heads;
  int best = 0;
  double best_cost = 1e300;
  for (int c = 1; c <= 16 && c <= tiles; ++c) {
    const int ct = (tiles + c - 1) / c;
    if (ct > cap) continue;
    const double fills = ct <= S ? 2.0 * ct : 3.0 * ct - S;
    const long long ctas = work * c;
    const int slots = slots_of(c, ct);
    if (slots <= 0) continue;
    const double waves = (double)((ctas + slots - 1) / slots);
    const double cost = waves * (fills + ovh);
    if (cost < best_cost * 0.98) best_cost = cost, best = c;
  }
  if (force_c >= 1 && force_c <= 16 && (tiles + force_c - 1) / force_c <= cap) best = force_c;
  if (best == 0) return false;
  *C_out = best;
  *chunk_out = ((tiles + best - 1) / best) * TK;
  return true;
}

// TMA descriptors of one layer's K or V pool: [slots][kv heads][128] bf16, 16 x 1 x 64 boxes,
// SWIZZLE_128B (the UMMA K-major tile layout); cached per (base, slots, heads)
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
static bool pool_map(CUtensorMap* out, const void* base, int64_t slots, int kv_heads) {
  static std::mutex mu;
  static EncodeTiledFn encode = nullptr;
  static std::map<std::tuple<uintptr_t, int64_t, int>, CUtensorMap> cache;
  std::lock_guard<std::mutex> lock(mu);
  const auto key = std::make_tuple(reinterpret_cast<uintptr_t>(base), slots, kv_heads);
  auto it = cache.find(key);
  if (it != cache.end()) {
    *out = it->second;
    return true;
  }
  if (encode == nullptr) {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess || fn == nullptr) {
      cudaGetLastError();
      return false;
    }
    encode = reinterpret_cast<EncodeTiledFn>(fn);
  }
  const cuuint64_t dims[3] = {(cuuint64_t)umma_attn::D, (cuuint64_t)kv_heads, (cuuint64_t)slots};
  const cuuint64_t strides[2] = {(cuuint64_t)umma_attn::D * 2, (cuuint64_t)kv_heads * umma_attn::D * 2};
  const cuuint32_t box[3] = {64, 1, 16};
  const cuuint32_t estr[3] = {1, 1, 1};
  CUtensorMap m;
  if (encode(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(base), dims, strides, box, estr,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return false;
  if (cache.size() > 4096) cache.clear();
  cache[key] = m;
  *out = m;
  return true;
}

struct UmmaPlan {
  int NR, C, chunk;
};

// Verify-kernel plan: NR = query rows rounded up to 8 (<= 80); two CTAs per SM up to NR = 48.
static bool umma_plan(const sd_paged_kv* kvp, int num_items, int max_keys, int max_nq, int q_heads, int dense,
                      UmmaPlan* pl) {
  using namespace umma_attn;
  const int G = q_heads / kvp->kv_heads;
  if (kvp->dtype != SD_DTYPE_BF16 || kvp->head_dim != D) return false;
  if (!(G == 4 || G == 8)) return false;
  const int NR = (max_nq * G + 7) & ~7;
  if (NR > kMaxNR) return false;
  const bool narrow = NR <= kNarrowMaxNR;
  const int tcols = narrow ? 256 : 512, nslot = narrow ? 2 : 4;
  const int S = tcols / NR;
  const int cap = chunk_cap_tiles(NR, nslot, S, narrow ? 113 * 1024 : 227 * 1024, dense);
  int C = 1, chunk = TK;
  // CTA slots for C-CTA clusters.  Clusters live inside one GPC, so sizes that do not tile
  // a GPC's slots leave some idle: the cluster-occupancy API gives that packing (it counts
  // one CTA per SM for this kernel although two are resident — ncu: occupancy limit 2 —
  // so it is doubled).  C = 1, 2, 4 pack every SM's two slots (C sweeps at ctx 4K / 16K and
  // at bench.py's 25-item launch, profiles/r2_cluster_sweep.md).
  const int per_sm = narrow ? 2 : 1;
  auto slots_of = [&](int c, int ct) -> int {
    if (c == 1 || c == 2 || c == 4) return 148 * per_sm;
    static std::mutex mu;
    static std::map<std::tuple<int, int, int, int, int>, int> cache;
    const int smem = make_layout(NR, nslot, S, ct, dense).total;
    const auto key = std::make_tuple(G, NR, c, smem, dense);
    std::lock_guard<std::mutex> lock(mu);
    auto itc = cache.find(key);
    if (itc != cache.end()) return itc->second;
    int v = G == 4 ? verify_slots_g4(NR, c, smem) : verify_slots_g8(NR, c, smem);
    v = std::min(148 * per_sm, std::max(0, v) * per_sm);
    cache[key] = v;
    return v;
  };
  if (cap == 0 || !plan_umma(max_keys < 1 ? 1 : max_keys, num_items, kvp->kv_heads, S, cap, slots_of, &C, &chunk,
                             dense))
    return false;
  pl->NR = NR, pl->C = C, pl->chunk = chunk;
  static const int log_plan = env_int("SD_ATTN_PLAN_LOG", 0);
  if (log_plan > 1) {
    static bool once = false;
    if (!once) {
      once = true;
      for (int c = 1; c <= 16; ++c)
        for (int ct : {1, 8, 32})
          fprintf(stderr, "[sd slots] G=%d NR=%d C=%d ct=%d slots=%d\n", G, NR, c, ct, slots_of(c, ct));
    }
  }
  if (log_plan)
    fprintf(stderr, "[sd plan] items=%d keys=%d NR=%d C=%d chunk_tiles=%d slots=%d dense=%d\n", num_items, max_keys,
            NR, C, chunk / TK, slots_of(C, chunk / TK), dense);
  return true;
}

// The tcgen05 kernels cover every bf16 shape with head_dim 128, GQA 4 or 8 and at most
// 80 query rows per item (callers chunk longer windows); anything else runs the generic kernel.
bool umma_supported(const sd_paged_kv* kvp, int max_nq, int q_heads) {
  using namespace umma_attn;
  const int G = q_heads / kvp->kv_heads;
  return kvp->dtype == SD_DTYPE_BF16 && kvp->head_dim == D && (G == 4 || G == 8) && max_nq * G <= kMaxNR;
}

int launch_attn_umma(const void* q, void* out, float* lse, const sd_paged_kv* kvp, int layer, const int32_t* items,
                     int num_items, int max_keys, int max_nq, const int32_t* crit, unsigned long long* acc,
                     int64_t acc_stride, int acc_shift, const int32_t* planted, int n_planted, float bonus,
                     int q_heads, float scale, void* ws, int64_t ws_bytes, cudaStream_t stream, bool* handled) {
  using namespace umma_attn;
  *handled = false;
  Params prm{};
  prm.q = static_cast<const __nv_bfloat16*>(q);
  prm.out = static_cast<__nv_bfloat16*>(out);
  prm.lse_out = lse;
  prm.kv = make_paged(kvp);
  prm.layer = layer;
  prm.items = items;
  prm.crit = crit;
  prm.acc = acc;
  prm.acc_stride = acc_stride;
  prm.acc_scale = ldexpf(1.f, acc_shift);
  prm.planted = planted;
  prm.n_planted = n_planted;
  prm.bonus_log2 = bonus * LOG2E;
  prm.q_heads = q_heads;
  prm.scale_log2 = scale * LOG2E;
  const int G = q_heads / kvp->kv_heads;
  static const int trace = env_int("SD_ATTN_TRACE", 0);
  if (trace) {
    if (g_trace_buf == nullptr) cudaMalloc(&g_trace_buf, sizeof(uint64_t) * kTraceCtas * kTraceSlots);
    prm.trace = g_trace_buf;
  }
  static const int hp_env = env_int("SD_UMMA_HP", 1);
  if (hp_env && max_nq == 1 && kvp->dtype == SD_DTYPE_BF16 && kvp->head_dim == D && (G == 4 || G == 8) &&
      kvp->kv_heads % 4 == 0) {
    // K1: 4 heads per CTA, 32 keys per tile, the whole key list in one CTA
    const int NR = 4 * G, tmax = (256 - NR) / NR;
    const int ct_tiles = (max(max_keys, 1) + 31) / 32;      // 32-key tiles
    const int ct = (ct_tiles * 32 + TK - 1) / TK;           // 128-key units for the staging arrays
    if (ct_tiles <= tmax && make_hp_layout(NR, 2, tmax, ct).total <= 113 * 1024) {  // logits stay resident
      prm.chunk = ct * TK;
      *handled = true;
      // a third 32 KB ring slot when two CTAs per SM still fit (deeper loads in flight)
      static const int hp_slots = env_int("SD_UMMA_HP_SLOTS", 3);
      const bool three = hp_slots == 3 && make_hp_layout(NR, 3, tmax, ct).total <= 113 * 1024;
      if (G == 4)
        return three ? launch_hp<4, 4, 3, 256>(prm, num_items, kvp->kv_heads, ct, stream)
                     : launch_hp<4, 4, 2, 256>(prm, num_items, kvp->kv_heads, ct, stream);
      return three ? launch_hp<8, 4, 3, 256>(prm, num_items, kvp->kv_heads, ct, stream)
                   : launch_hp<8, 4, 2, 256>(prm, num_items, kvp->kv_heads, ct, stream);
    }
  }
  const int dense = (crit == nullptr && kvp->page_shift >= 4) ? 1 : 0;
  static const int tma_env = env_int("SD_K2_TMA", 1);
  if (dense && tma_env) {  // dense K2 chunks stream through TMA boxes (one descriptor per pool and layer)
    const int64_t loff = (int64_t)layer * kvp->layer_stride * 2;  // bytes (bf16)
    prm.tma = pool_map(&prm.tmk, static_cast<const char*>(kvp->k) + loff, kvp->num_slots, kvp->kv_heads) &&
              pool_map(&prm.tmv, static_cast<const char*>(kvp->v) + loff, kvp->num_slots, kvp->kv_heads);
  }
  UmmaPlan pl;
  if (!umma_plan(kvp, num_items, max_keys, max_nq, q_heads, dense, &pl)) return 0;
  prm.chunk = pl.chunk;
  prm.dense = dense;
  *handled = true;
  return G == 4 ? launch_verify_g4(prm, pl.NR, pl.C, num_items, kvp->kv_heads, stream)
                : launch_verify_g8(prm, pl.NR, pl.C, num_items, kvp->kv_heads, stream);
}

}  // namespace sd

// Diagnostics: per-CTA phase timestamps of the last traced verify launch (SD_ATTN_TRACE=1):
// [ctas][12] uint64 = start, setup done, phase 1 done, lse known, phase 2 done, O ready,
// end, producer done, -, smid | tiles << 32.
extern "C" int sd_attention_trace_umma(uint64_t* host_dst, int32_t ctas) {
  if (ctas > sd::umma_attn::kTraceCtas) ctas = sd::umma_attn::kTraceCtas;
  if (sd::umma_attn::g_trace_buf == nullptr) return -1;
  cudaError_t e = cudaMemcpy(host_dst, sd::umma_attn::g_trace_buf, sizeof(uint64_t) * sd::umma_attn::kTraceSlots * ctas,
                             cudaMemcpyDeviceToHost);
  return e == cudaSuccess ? 0 : (int)e;
}
