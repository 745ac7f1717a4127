// tcgen05 (UMMA) paged attention for sm_100a: K2 verify with PillarAttn score
// emission, every K and V row read from HBM exactly once while the item's key
// chunk fits the TMEM-resident logits.
//
// Orientation ("swap AB"): the KEYS of a 128-key tile are the UMMA M dimension
// and the item's query rows (token x GQA group, padded to NR = a multiple of 8,
// 8..80) are N:
//
//   S^T[128 keys][NR] = K_tile[128][d] . Q^T            (kind::f16, K = d)
//   O^T[d][NR]       += V_tile^T[d][128] . P^T[128][NR]  (A MN-major, K = keys)
//
// so TMEM lane = key (phase 1/2) and lane = head-dim column (epilogue): each
// softmax thread owns ONE key and holds the NR query-row logits of it.
// Consequences:
//   * per-row online (max, sum) is thread-local across tiles; the cross-key
//     reduction happens once per CTA (shuffles + smem + DSMEM across the
//     cluster), not once per tile;
//   * the PillarAttn score  acc[token][pos] += sum_g exp(s - lse)  is a
//     register-local sum over the G group columns: one RED per (key, token),
//     in 64-bit fixed point so the accumulation order cannot change the sum;
//   * the planted bonus and the causal mask are per-key scalars.
//
// TMEM holds S = TCOLS / NR slots of NR fp32 columns.  Slot S-1 doubles as the
// O^T accumulator: phase 2 first consumes the tile whose logits sit there, and
// the first PV MMA (which overwrites those columns) waits for that read.  So a
// chunk of up to S tiles keeps all its logits in TMEM between the passes (the
// exact lse is known before any probability is formed, SURVEY.md §7.2 option
// (c)) and K is read once; longer chunks recompute the evicted tiles' logits in
// phase 2 (K re-read for those tiles only, V still once).
//
//   grid = (C, kv_heads, items), cluster (C,1,1): CTA c owns keys
//   [c*chunk, (c+1)*chunk) of the item's key list (critical list, then the
//   dense causal range).
//   warps 0-3  softmax / scores / P^T -> smem / epilogue (TMEM lanes 0..127)
//   warp 4     producer: 16-byte cp.async of 256-byte key rows (paged gather)
//              into an NSLOT x 32 KB ring in the UMMA SWIZZLE_128B layout
//   warp 5     TMEM allocator + single-thread tcgen05.mma issuer
//
// Restates model.py:229-253 (_attend) for forward_full (model.py:318-334) and
// forward_sparse (model.py:360-380), and the score path selection.py:78-135.
#pragma once
#include "umma_common.cuh"

namespace sd {
namespace umma_attn {

constexpr uint32_t kNoTmem = 0xffffffffu;

// TMEM columns loaded per step by the softmax warps (bounds live registers at large NR)
template <int NR>
constexpr int col_chunk() {
  return NR <= 40 ? NR : NR % 32 == 0 ? 32 : NR % 24 == 0 ? 24 : NR % 16 == 0 ? 16 : 8;
}

// Tile schedule shared by the producer, the MMA issuer and the softmax warps.
//   phase 1: K tiles 0..nt-1, logits of tile t into slot t % S (use t / S)
//   phase 2: the resident tiles [nt-TR, nt) — the one in the O slot (S-1) first — then
//            the evicted tiles 0..E-1, whose logits are recomputed into slots 0..S-2
struct Sched {
  int nt, S, TR, E, t_o;
  __device__ __forceinline__ Sched(int nt_, int S_) : nt(nt_), S(S_) {
    TR = min(nt, S);
    E = nt - TR;
    t_o = -1;
    if (nt >= S) t_o = (nt - 1) - ((nt - 1 - (S - 1)) % S);  // largest t < nt with t % S == S-1
  }
  __device__ __forceinline__ int p2_tile(int i2) const {
    if (i2 >= TR) return i2 - TR;
    if (t_o < 0) return i2;
    if (i2 == 0) return t_o;
    const int t = nt - S + (i2 - 1);
    return t >= t_o ? t + 1 : t;
  }
  __device__ __forceinline__ int uses1(int j) const { return nt > j ? (nt - 1 - j) / S + 1 : 0; }
  __device__ __forceinline__ void p2_slot(int i2, int& slot, int& use) const {
    if (i2 < TR) {
      const int t = p2_tile(i2);
      slot = t % S, use = t / S;
      return;
    }
    const int k = i2 - TR;
    slot = k % (S - 1);
    use = uses1(slot) + k / (S - 1);
  }
  // producer ring fill f -> (tile, K or V)
  __device__ __forceinline__ void fill(int f, int& t, bool& isv) const {
    if (f < nt) {
      t = f, isv = false;
    } else if (f < nt + TR) {
      t = p2_tile(f - nt), isv = true;
    } else {
      const int g = f - nt - TR;
      t = g >> 1, isv = g & 1;
    }
  }
  __device__ __forceinline__ int nfill() const { return 3 * nt - TR; }
};

// Row statistics of NR rows (m, l in registers, one key per lane) reduced over the warp in
// blocks of 32 / 16 / 8 rows; lane L of a block of size BS ends up with row B0 + (L % BS).
template <int NR, int B0>
__device__ __forceinline__ void rows_reduce_store(float* m, float* l, int lane, int warp, int R, float* wm, float* wl) {
  if constexpr (B0 < NR) {
    constexpr int BS = NR - B0 >= 32 ? 32 : NR - B0 >= 16 ? 16 : 8;
    warp_rows_reduce<BS>(m + B0, l + B0, lane);
    const int row = B0 + (lane & (BS - 1));
    if (lane < BS && row < R) wm[warp * NR + row] = m[B0], wl[warp * NR + row] = l[B0];
    rows_reduce_store<NR, B0 + BS>(m, l, lane, warp, R, wm, wl);
  }
}

template <int G, int NR, int NSLOT, int TCOLS>
// ext_tmem: a TMEM base the caller allocated (the fused kernel), or kNoTmem to allocate here
__device__ __forceinline__ void verify_body(const Params& p, const int h, const int item_idx, uint32_t ext_tmem = kNoTmem) {
  constexpr int S = TCOLS / NR;             // logits slots (slot S-1 = O^T accumulator)
  constexpr int OCOL = (S - 1) * NR;
  constexpr int CH = col_chunk<NR>();
  static_assert(NR % 8 == 0 && NR % G == 0 && S >= 2 && CH % G == 0, "verify tile shape");

  cg::cluster_group cluster = cg::this_cluster();
  const int C = static_cast<int>(cluster.num_blocks());
  const int crank = static_cast<int>(cluster.block_rank());
  const Item it = load_item(p.items, item_idx);
  const int R = it.nq * G;
  const int Nk = it.num_keys();
  // the item's key tiles split evenly over the cluster (counts differ by at most one; the
  // partial last tile goes to the last CTA, which then streams one mostly empty tile more
  // than its peers instead of a whole chunk's worth of peers waiting for it); at most
  // p.chunk / TK tiles per CTA as the planner sized them
  const int kt = (Nk + TK - 1) / TK;
  const int kb = (crank * kt / C) * TK;
  const int ke = min(Nk, ((crank + 1) * kt / C) * TK);
  const int nk = max(0, ke - kb);
  const Sched sc((nk + TK - 1) / TK, S);
  const int nt = sc.nt;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int cta_lin = (blockIdx.z * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x;
#define TRACE(k, val)                                                                                   \
  do {                                                                                                  \
    if (p.trace && cta_lin < kTraceCtas) p.trace[cta_lin * kTraceSlots + (k)] = (val);                  \
  } while (0)
  if (tid == 0) {
    uint32_t smid;
    asm volatile("mov.u32 %0, %smid;" : "=r"(smid));
    TRACE(0, gtime());
    TRACE(9, (uint64_t)smid | ((uint64_t)nt << 32));
  }

  extern __shared__ unsigned char smem_raw[];
  unsigned char* smem = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const Layout L = make_layout(NR, NSLOT, S, p.chunk / TK, p.dense);
  unsigned char* ring = smem + L.ring;
  unsigned char* qs = smem + L.q;
  unsigned char* pbuf = smem + L.pbuf;
  int32_t* spos = reinterpret_cast<int32_t*>(smem + L.pos);
  int32_t* sslot = reinterpret_cast<int32_t*>(smem + L.slot);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + L.bar);
  uint64_t* empty = full + NSLOT;
  uint64_t* sfull = empty + NSLOT;       // [S] logits of the slot's current use are in TMEM
  uint64_t* sfree = sfull + S;           // [S] softmax warps are done reading the slot
  uint64_t* pready = sfree + S;          // [2] P^T buffer written
  uint64_t* pfree = pready + 2;          // [2] P^T buffer consumed by the PV MMA
  uint64_t* obar = pfree + 2;            // O^T complete
  uint64_t* qbar = obar + 1;             // the Q tile is in shared memory (softmax warps wrote it)
  float* wm = reinterpret_cast<float*>(smem + L.wm);
  float* wl = reinterpret_cast<float*>(smem + L.wl);
  float* xm = reinterpret_cast<float*>(smem + L.xm);
  float* xl = reinterpret_cast<float*>(smem + L.xl);
  float* rowlse = reinterpret_cast<float*>(smem + L.rowlse);
  uint32_t* tptr = reinterpret_cast<uint32_t*>(smem + L.tptr);

  // dense chunks starting on a 16-key boundary stream through TMA boxes of 16 keys (producer
  // lanes 0-7 issue the two 64-element halves of one box each); otherwise 16-byte cp.async
  const bool use_tma = p.tma && p.dense && ((it.dense_lo + kb) & 15) == 0;

  // ---- setup ----
  if (warp == WMMA && ext_tmem == kNoTmem) tmem_alloc(tptr, TCOLS);
  if (tid == 0) {
    // TMA fills: one arrival with the transaction bytes; cp.async fills: one per producer lane
    for (int i = 0; i < NSLOT; ++i) mbar_init(full + i, use_tma ? 1 : 32), mbar_init(empty + i, 1);
    for (int i = 0; i < S; ++i) mbar_init(sfull + i, 1), mbar_init(sfree + i, NSW);
    mbar_init(pready + 0, NSW), mbar_init(pready + 1, NSW);
    mbar_init(pfree + 0, 1), mbar_init(pfree + 1, 1);
    mbar_init(obar, 1);
    mbar_init(qbar, NSW);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  // key positions and their physical slots for the whole chunk (the producer's copy loop
  // then never waits on a block-table load); keys past the chunk copy the last valid row
  // (finite data, masked out of the softmax).  Dense items stage only the page ids, and the
  // producer warp does that itself after the CTA barrier (its first TMA boxes do not wait
  // for the Q tile, which the softmax warps load meanwhile).
  const int32_t* trow = p.kv.table + (int64_t)it.table_row * p.kv.table_stride;
  const int pshift = p.kv.page_shift, pmask = (1 << pshift) - 1;
  const int dpos0 = it.dense_lo + kb;          // dense: position of chunk key 0
  const int dpage0 = dpos0 >> pshift;
  int32_t* spage = spos;                       // dense: [page - dpage0] -> physical page
  if (!p.dense) {
    const int nkeys = nt * TK;
    for (int j0 = 0; j0 < nkeys; j0 += 8 * NT) {  // 8 independent loads in flight per thread
      int pos[8], pg[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) pos[k] = it.key_pos(p.crit, min(kb + j0 + k * NT + tid, ke - 1));
#pragma unroll
      for (int k = 0; k < 8; ++k) pg[k] = __ldg(trow + (pos[k] >> pshift));
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const int j = j0 + k * NT + tid;
        if (j < nkeys) {
          spos[j] = kb + j < ke ? pos[k] : -1;
          sslot[j] = (pg[k] << pshift) | (pos[k] & pmask);
        }
      }
    }
  }
  // chunk-relative key j -> absolute position (-1 past the chunk) / physical slot
  auto pos_of = [&](int j) -> int {
    if (p.dense) return kb + j < ke ? dpos0 + j : -1;
    return spos[j];
  };
  auto slot_of = [&](int j) -> int {
    if (!p.dense) return sslot[j];
    const int pos = it.dense_lo + min(kb + j, ke - 1);
    return (spage[(pos >> pshift) - dpage0] << pshift) | (pos & pmask);
  };
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = ext_tmem == kNoTmem ? *tptr : ext_tmem;
  if (warp < NSW) {
    // Q rows (token-major: r = tok*G + g) -> [dhalf][NR][128 B] SWIZZLE_128B, zero padding rows
    for (int i = tid; i < NR * 16; i += NSW * 32) {
      const int r = i >> 4, c = i & 15;
      uint4 v = make_uint4(0, 0, 0, 0);
      if (r < R)
        v = *reinterpret_cast<const uint4*>(p.q + ((int64_t)(it.q_row0 + r / G) * p.q_heads + h * G + r % G) * D +
                                            c * 8);
      *reinterpret_cast<uint4*>(qs + (c >> 3) * (NR * 128) + r * 128 + (((c & 7) ^ (r & 7)) << 4)) = v;
    }
    fence_proxy_async();
    __syncwarp();
    if (lane == 0) mbar_arrive(qbar);
  } else if (warp == WPROD && p.dense && nk > 0) {
    const int lastpg = (it.dense_lo + ke - 1) >> pshift;
    const int npg = ((dpos0 + nt * TK - 1) >> pshift) - dpage0 + 1;
    for (int i = lane; i < npg; i += 32) spage[i] = __ldg(trow + min(dpage0 + i, lastpg));
    __syncwarp();
  }
  if (tid == 0) TRACE(1, gtime());
  // barrier 0 (C > 1): every peer of the cluster has started before anyone touches its shared
  // memory (the statistics push below); arrived here, waited right before the first DSMEM use
  if (C > 1) asm volatile("barrier.cluster.arrive.relaxed.aligned;\n" ::: "memory");

  const int64_t row_stride = (int64_t)p.kv.kv_heads * D;  // elements between consecutive slots
  const __nv_bfloat16* Kg = static_cast<const __nv_bfloat16*>(p.kv.k) + (int64_t)p.layer * p.kv.layer_stride + h * D;
  const __nv_bfloat16* Vg = static_cast<const __nv_bfloat16*>(p.kv.v) + (int64_t)p.layer * p.kv.layer_stride + h * D;

  if (warp == WPROD) {
    // ===================== producer =====================
    const uint64_t pol = policy_evict_first();  // every row is read once (K of evicted tiles twice)
    const int sub = lane >> 4, c = lane & 15;   // 2 key rows x 16 chunks per instruction
    const uint32_t ring_u = smem_u32(ring);
    const int nfill = sc.nfill();
    for (int f = 0; f < nfill; ++f) {
      const int s = f % NSLOT;
      int t;
      bool isv;
      sc.fill(f, t, isv);
      const uint32_t tile_u = ring_u + s * TILE_BYTES;
      if (use_tma) {
        int slot0 = 0;
        if (lane < TK / 16) {
          const int pos = it.dense_lo + min(kb + t * TK + lane * 16, ke - 1);
          slot0 = ((spage[(pos >> pshift) - dpage0] << pshift) | (pos & pmask)) & ~15;
        }
        if (f >= NSLOT) mbar_wait(empty + s, ((f / NSLOT) - 1) & 1);
        if (lane < TK / 16) {
          const CUtensorMap* map = isv ? &p.tmv : &p.tmk;
          tma_box(tile_u + lane * 2048, map, 0, h, slot0, full + s, pol);
          tma_box(tile_u + TK * 128 + lane * 2048, map, 64, h, slot0, full + s, pol);
        }
        __syncwarp();
        if (lane == 0) mbar_arrive_tx(full + s, TILE_BYTES);
      } else {
        const __nv_bfloat16* base = (isv ? Vg : Kg) + c * 8;
        int sl[4];  // physical slots of keys lane + 32m, broadcast by shuffles below
#pragma unroll
        for (int m = 0; m < 4; ++m) sl[m] = slot_of(t * TK + m * 32 + lane);
        if (f >= NSLOT) mbar_wait(empty + s, ((f / NSLOT) - 1) & 1);
        const uint32_t dst0 = tile_u + (c >> 3) * (TK * 128);
#pragma unroll
        for (int kk = 0; kk < TK / 2; ++kk) {
          const int i = 2 * kk + sub;  // key row within the tile
          const int slot = __shfl_sync(0xffffffffu, sl[kk >> 4], i & 31);
          cp_async16(dst0 + i * 128 + (((c & 7) ^ (i & 7)) << 4), base + (int64_t)slot * row_stride, pol);
        }
        cp_async_mbar_arrive(full + s);
      }
      if (f == nt - 1) {
        if (lane == 0) TRACE(11, gtime());
        if (C > 1) {
          cluster_wait();    // barrier 0
          cluster_arrive();  // barrier 1: K streamed; let the exchange proceed
        }
      }
    }
    if (lane == 0) TRACE(7, gtime());
    if (C > 1) {
      if (nt == 0) {
        cluster_wait();  // barrier 0
        cluster_arrive();
      }
      cluster_wait();
      for (int b = 0; b < 2; ++b) {  // the softmax warps' epilogue barriers
        cluster_arrive();
        cluster_wait();
      }
    }
    return;
  }

  if (warp == WMMA) {
    // ===================== MMA issuer =====================
    const uint32_t ring_u = smem_u32(ring), q_u = smem_u32(qs), p_u = smem_u32(pbuf);
    const uint32_t id_qk = idesc_bf16(NR, false, false);
    const uint32_t id_pv = idesc_bf16(NR, true, true);
    const bool leader = lane == 0;
    int f = 0;
    mbar_wait(qbar, 0);
    // S^T of one tile into TMEM slot `slot` (its use-th occupant) from the next ring fill
    auto qk = [&](int slot, int use) {
      const int s = f % NSLOT;
      mbar_wait(full + s, (f / NSLOT) & 1);
      if (use > 0) mbar_wait(sfree + slot, (use - 1) & 1);
      fence_proxy_async();
      tc_fence_after();
      if (leader) {
        const uint32_t a0 = ring_u + s * TILE_BYTES;
#pragma unroll
        for (int ks = 0; ks < D / 16; ++ks) {
          const uint32_t off = (ks & 3) << 5;  // K = 16 bf16 = 32 B steps inside the 128-B atom
          const uint64_t a = smem_desc(a0 + (ks >> 2) * (TK * 128) + off, 16, 1024, 2);
          const uint64_t b = smem_desc(q_u + (ks >> 2) * (NR * 128) + off, 16, 1024, 2);
          umma(tbase + slot * NR, a, b, id_qk, ks > 0);
        }
        umma_commit(empty + s);
        umma_commit(sfull + slot);
      }
      __syncwarp();
      ++f;
    };
    for (int t = 0; t < nt; ++t) qk(t % S, t / S);
    if (lane == 0) TRACE(10, gtime());
    if (C > 1) {
      cluster_wait();    // barrier 0
      cluster_arrive();  // barrier 1: this warp's part of phase 1 is issued
    }
    for (int i2 = 0; i2 < nt; ++i2) {
      if (i2 >= sc.TR) {  // evicted tile: recompute its logits
        int slot, use;
        sc.p2_slot(i2, slot, use);
        qk(slot, use);
      }
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
          // A = V^T: MN-major SW128, 64-d atoms LBO = 16 KB apart, 8-key groups SBO = 1 KB
          const uint64_t a = smem_desc(a0 + ks * 16 * 128, TK * 128, 1024, 2);
          // B = P^T: MN-major no swizzle, 8-key core groups LBO = 128 B, 8-row groups SBO = 2 KB
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
    if (C > 1) {
      cluster_wait();
      for (int b = 0; b < 2; ++b) {  // the softmax warps' epilogue barriers
        cluster_arrive();
        cluster_wait();
      }
    }
    asm volatile("bar.sync 2, %0;\n" ::"n"((NSW + 1) * 32) : "memory");  // softmax warps read O
    tc_fence_after();
    if (ext_tmem == kNoTmem) tmem_dealloc(tbase, TCOLS);
    return;
  }

  // ===================== softmax warps (TMEM lane = key) =====================
  const int kl = warp * 32 + lane;                  // key (and later d) index within the tile
  const uint32_t tl = tbase + ((uint32_t)(warp * 32) << 16);
  float m[NR], l[NR];
#pragma unroll
  for (int r = 0; r < NR; ++r) m[r] = -INFINITY, l[r] = 0.f;

  // per-key scalars for tile t: position, bias and first visible row (rows >= rmin see the key)
  auto key_info = [&](int t, int& pos, float& bias, int& rmin) {
    const int j = t * TK + kl;
    pos = pos_of(j);
    if (pos < 0) {
      rmin = NR;  // past the chunk: invisible to every row
      bias = 0.f;
      return;
    }
    rmin = kb + j < it.crit_len ? 0 : max(0, pos - it.qpos0) * G;
    bias = p.n_planted ? planted_bias(p.planted, p.n_planted, p.bonus_log2, pos) : 0.f;
  };
  auto release = [&](int slot) {  // one elected arrival per warp
    tc_fence_before();
    __syncwarp();
    if (lane == 0) mbar_arrive(sfree + slot);
  };

  // ---- phase 1: S^T tiles -> thread-local online (max, sum) ----
  for (int t = 0; t < nt; ++t) {
    int pos, rmin;
    float bias;
    key_info(t, pos, bias, rmin);
    const int slot = t % S;
    mbar_wait(sfull + slot, (t / S) & 1);
    tc_fence_after();
#pragma unroll
    for (int c0 = 0; c0 < NR; c0 += CH) {
      float v[CH];
      tmem_ld_cols<CH>(tl + slot * NR + c0, v);
      tmem_wait_ld();
      if (c0 + CH >= NR && t < sc.E) release(slot);  // evicted before phase 2: recomputed there
#pragma unroll
      for (int i = 0; i < CH; ++i) {
        const int r = c0 + i;
        if (r >= rmin && r < R) {
          const float s2 = fmaf(v[i], p.scale_log2, bias);
          const float nm = fmaxf(m[r], s2);
          l[r] = l[r] * ex2(m[r] - nm) + ex2(s2 - nm);
          m[r] = nm;
        }
      }
    }
  }
  if (tid == 0) TRACE(2, gtime());
  // ---- exchange: warp -> CTA -> cluster row statistics -> exact lse ----
  rows_reduce_store<NR, 0>(m, l, lane, warp, R, wm, wl);
  sw_bar();
  if (C > 1) cluster_wait();  // barrier 0: all peers have started (DSMEM pushes follow)
  if (tid < R) {
    float mm = -INFINITY, ll = 0.f;
#pragma unroll
    for (int w = 0; w < NSW; ++w) {
      const float om = wm[w * NR + tid], ol = wl[w * NR + tid];
      const float nm = fmaxf(mm, om);
      ll = (nm == -INFINITY) ? 0.f : ll * ex2(mm - nm) + ol * ex2(om - nm);
      mm = nm;
    }
    // push this CTA's row statistics into every peer's [crank][row] slot (remote
    // stores are fire-and-forget; the cluster barrier's release/acquire orders them)
    for (int c = 0; c < C; ++c) {
      *cluster.map_shared_rank(xm + crank * NR + tid, c) = mm;
      *cluster.map_shared_rank(xl + crank * NR + tid, c) = ll;
    }
  }
  if (tid == 0) TRACE(8, gtime());
  if (C > 1) {
    cluster_arrive();
    cluster_wait();
  } else {
    sw_bar();
  }
  if (tid < NR) {
    float lse2 = INFINITY;  // padding rows -> P = 0
    if (tid < R) {
      float M = -INFINITY;
      for (int c = 0; c < C; ++c) M = fmaxf(M, xm[c * NR + tid]);
      float Ls = 0.f;
      for (int c = 0; c < C; ++c) {
        const float mc = xm[c * NR + tid];
        if (mc != -INFINITY) Ls += xl[c * NR + tid] * ex2(mc - M);
      }
      lse2 = M + log2f(Ls);
    }
    rowlse[tid] = lse2;
  }
  sw_bar();
  if (tid == 0) TRACE(3, gtime());

  // ---- phase 2: P = exp2(S - lse) (final), scores, P^T -> smem for the PV MMA ----
  const bool scores = p.acc != nullptr && it.acc_row >= 0;
  unsigned long long* acc_base = scores ? p.acc + (int64_t)it.acc_row * p.acc_stride : nullptr;
  const int64_t acc_tok_stride = (int64_t)it.acc_step * p.acc_stride;
  for (int i2 = 0; i2 < nt; ++i2) {
    const int t = sc.p2_tile(i2);
    int slot, use;
    sc.p2_slot(i2, slot, use);
    int pos, rmin;
    float bias;
    key_info(t, pos, bias, rmin);
    mbar_wait(sfull + slot, use & 1);
    tc_fence_after();
    if (i2 >= 2) mbar_wait(pfree + (i2 & 1), ((i2 >> 1) - 1) & 1);
    // P^T [key][row]: core matrix (8 keys x 8 rows) = 128 B; key groups 128 B apart,
    // row groups TK*16 B apart -> this thread's 8-row chunks at kl*16 + ng*TK*16
    unsigned char* pb = pbuf + (i2 & 1) * (NR * TK * 2) + kl * 16;
    const bool live = scores && rmin < R;
    float sum_all = 0.f;
#pragma unroll
    for (int c0 = 0; c0 < NR; c0 += CH) {
      float v[CH];
      tmem_ld_cols<CH>(tl + slot * NR + c0, v);
      tmem_wait_ld();
      if (c0 + CH >= NR) release(slot);
#pragma unroll
      for (int i = 0; i < CH; ++i) {
        const int r = c0 + i;
        v[i] = (r >= rmin && r < R) ? ex2(fmaf(v[i], p.scale_log2, bias) - rowlse[r]) : 0.f;
      }
      if (live) {
        if (it.acc_step == 0) {
#pragma unroll
          for (int i = 0; i < CH; ++i) sum_all += v[i];
        } else {
#pragma unroll
          for (int tk = 0; tk < CH / G; ++tk) {
            float sum = 0.f;
#pragma unroll
            for (int g = 0; g < G; ++g) sum += v[tk * G + g];
            if (sum != 0.f) red_add_fx(acc_base + (c0 / G + tk) * acc_tok_stride + pos, sum, p.acc_scale);
          }
        }
      }
#pragma unroll
      for (int ng = 0; ng < CH / 8; ++ng) {
        __nv_bfloat162 b0 = __floats2bfloat162_rn(v[ng * 8 + 0], v[ng * 8 + 1]);
        __nv_bfloat162 b1 = __floats2bfloat162_rn(v[ng * 8 + 2], v[ng * 8 + 3]);
        __nv_bfloat162 b2 = __floats2bfloat162_rn(v[ng * 8 + 4], v[ng * 8 + 5]);
        __nv_bfloat162 b3 = __floats2bfloat162_rn(v[ng * 8 + 6], v[ng * 8 + 7]);
        uint4 w;
        w.x = *reinterpret_cast<uint32_t*>(&b0);
        w.y = *reinterpret_cast<uint32_t*>(&b1);
        w.z = *reinterpret_cast<uint32_t*>(&b2);
        w.w = *reinterpret_cast<uint32_t*>(&b3);
        *reinterpret_cast<uint4*>(pb + (c0 / 8 + ng) * TK * 16) = w;
      }
    }
    if (live && it.acc_step == 0 && sum_all != 0.f) red_add_fx(acc_base + pos, sum_all, p.acc_scale);
    fence_proxy_async();
    __syncwarp();
    if (lane == 0) mbar_arrive(pready + (i2 & 1));
  }

  // ---- epilogue: O^T (lane = d) -> cluster reduction -> out ----
  if (tid == 0) TRACE(4, gtime());
  if (nt > 0) {
    mbar_wait(obar, 0);
    tc_fence_after();
    if (tid == 0) TRACE(5, gtime());
  }
  const int dcol = kl;
  float* Ob = reinterpret_cast<float*>(ring);  // [NR][D] O^T partial (C > 1); the ring is idle now
#pragma unroll
  for (int c0 = 0; c0 < NR; c0 += CH) {
    float o[CH];
    if (nt > 0) {
      tmem_ld_cols<CH>(tl + OCOL + c0, o);
      tmem_wait_ld();
    } else {
#pragma unroll
      for (int i = 0; i < CH; ++i) o[i] = 0.f;
    }
#pragma unroll
    for (int i = 0; i < CH; ++i) {
      const int r = c0 + i;
      if (r < R) {
        if (C == 1)
          p.out[((int64_t)(it.q_row0 + r / G) * p.q_heads + h * G + r % G) * D + dcol] = __float2bfloat16_rn(o[i]);
        else
          Ob[r * D + dcol] = o[i];
      }
    }
  }
  tc_fence_before();
  asm volatile("bar.arrive 2, %0;\n" ::"n"((NSW + 1) * 32) : "memory");  // O read: TMEM may be freed
  if (C > 1) {
    // all MMAs of this CTA are complete (obar): row r is summed over the cluster by CTA
    // r % C (DSMEM loads issued back to back)
    cluster_arrive();
    cluster_wait();
    for (int r = crank; r < R; r += C) {
      float part[16];
#pragma unroll
      for (int c = 0; c < 16; ++c) part[c] = c < C ? *cluster.map_shared_rank(Ob + r * D + dcol, c) : 0.f;
      float sum = 0.f;
#pragma unroll
      for (int c = 0; c < 16; ++c) sum += part[c];
      p.out[((int64_t)(it.q_row0 + r / G) * p.q_heads + h * G + r % G) * D + dcol] = __float2bfloat16_rn(sum);
    }
  }
  if (p.lse_out != nullptr && crank == 0 && tid < R)
    p.lse_out[(int64_t)(it.q_row0 + tid / G) * p.q_heads + h * G + tid % G] = rowlse[tid] * LN2;
  if (C > 1) {  // peers may still be reading this CTA's partial
    cluster_arrive();
    cluster_wait();
  }
  if (tid == 0) TRACE(6, gtime());
#undef TRACE
}

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
  L.wm = o;    o += NSW * 8 * 2 * 4;     // 64-key heads: the two warps' (m, l) per q head
  L.wl = L.xm = L.xl = L.rowlse = 0;
  L.total = align_up(o, 128) + 1024;
  return L;
}

// head-packed kernel warp layout: softmax warps 0-3, NPROD producer warps, the MMA warp
// (the standalone K1 kernel runs HP_NPROD = 4 producers; inside the fused verify + draft
// kernel it runs on the verify kernel's six warps with one)
constexpr int HP_NPROD = 4;
constexpr int HP_NT = (NSW + HP_NPROD + 1) * 32;

template <int G, int HPC, int NSLOT, int TCOLS, int NPROD = HP_NPROD>
__device__ __forceinline__ void draft_body(const Params& p, const int hgroup, const int item_idx, uint32_t ext_tmem = kNoTmem) {
  constexpr int HP_WPROD = NSW, HP_WMMA = NSW + NPROD;
  constexpr int BNT = (NSW + NPROD + 1) * 32;
  constexpr int NQ = HPC * G;                       // q heads of the CTA
  constexpr int NR = NQ < 16 ? 16 : NQ;             // UMMA N
  constexpr int KPT = TK / HPC;                     // keys per tile
  constexpr int TMAX = (TCOLS - NR) / NR;
  constexpr int OCOL = TMAX * NR;
  constexpr int WH = KPT >= 32 ? 1 : 32 / KPT;      // heads per warp (rows of a warp)
  static_assert(KPT == 16 || KPT == 32 || KPT == 64, "head packing: 2, 4 or 8 heads per CTA");

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

  if (warp == HP_WMMA && ext_tmem == kNoTmem) tmem_alloc(tptr, TCOLS);
  if (tid == 0) {
    for (int i = 0; i < NSLOT; ++i) mbar_init(full + i, 32 * NPROD), mbar_init(empty + i, 1);
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
    for (int j0 = 0; j0 < nkeys; j0 += 8 * BNT) {
      int pos[8], pg[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) pos[k] = it.key_pos(p.crit, min(j0 + k * BNT + tid, nk - 1));
#pragma unroll
      for (int k = 0; k < 8; ++k) pg[k] = __ldg(trow + (pos[k] >> p.kv.page_shift));
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const int j = j0 + k * BNT + tid;
        if (j < nkeys) {
          spos[j] = j < nk ? pos[k] : -1;
          sslot[j] = (pg[k] << p.kv.page_shift) | (pos[k] & pmask);
        }
      }
    }
  }
  // Q: the CTA's NQ q heads are contiguous in the row (heads h0.. x group)
  for (int i = tid; i < NR * 16; i += BNT) {
    const int r = i >> 4, c = i & 15;
    uint4 v = make_uint4(0, 0, 0, 0);
    if (r < NQ) v = *reinterpret_cast<const uint4*>(p.q + ((int64_t)it.q_row0 * p.q_heads + h0 * G + r) * D + c * 8);
    *reinterpret_cast<uint4*>(qs + (c >> 3) * (NR * 128) + r * 128 + (((c & 7) ^ (r & 7)) << 4)) = v;
  }
  // P^T buffers: off-diagonal blocks stay zero for the whole launch
  for (int i = tid; i < 2 * NR * TK * 2 / 16; i += BNT) reinterpret_cast<uint4*>(pbuf)[i] = make_uint4(0, 0, 0, 0);
  fence_proxy_async();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = ext_tmem == kNoTmem ? *tptr : ext_tmem;
  if (tid == 0) HTRACE(1, gtime());

  const int64_t row_stride = (int64_t)p.kv.kv_heads * D;
  const __nv_bfloat16* Kg = static_cast<const __nv_bfloat16*>(p.kv.k) + (int64_t)p.layer * p.kv.layer_stride + h0 * D;
  const __nv_bfloat16* Vg = static_cast<const __nv_bfloat16*>(p.kv.v) + (int64_t)p.layer * p.kv.layer_stride + h0 * D;

  if (warp >= HP_WPROD && warp < HP_WPROD + NPROD) {
    // producers: warp pw copies rows [pw * 128 / NPROD, ...) of every 32 KB fill (one head's keys)
    const int pw = warp - HP_WPROD;
    const uint64_t pol = policy_evict_first();
    const int sub = lane >> 4, c = lane & 15;
    const uint32_t ring_u = smem_u32(ring);
    constexpr int KK = TK / 2 / NPROD;  // row pairs per warp
    for (int f = 0; f < nfill; ++f) {
      const int s = f % NSLOT;
      int t;
      bool isv;
      fill_tile_hp(f, nt, TR, t, isv);
      const __nv_bfloat16* base = (isv ? Vg : Kg) + c * 8;
      // physical slots of the tile's keys: lane L holds key L (and L + 32 for 64-key heads)
      const int sl = sslot[t * KPT + (lane % (KPT < 32 ? KPT : 32))];
      const int sl_hi = KPT == 64 ? sslot[t * KPT + 32 + lane] : 0;
      if (f >= NSLOT) mbar_wait(empty + s, ((f / NSLOT) - 1) & 1);
      const uint32_t dst0 = ring_u + s * TILE_BYTES + (c >> 3) * (TK * 128);
#pragma unroll
      for (int k2 = 0; k2 < KK; ++k2) {
        const int kk = pw * KK + k2;
        const int i = 2 * kk + sub;            // tile row = head-major (hh, key)
        const int hh = (2 * kk) / KPT;         // same for both rows of the instruction
        const int kin = (2 * kk) % KPT;          // even: both rows' keys lie in one 32-key half
        const int slot = __shfl_sync(0xffffffffu, KPT == 64 && kin >= 32 ? sl_hi : sl, (kin & 31) + sub);
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
    if (ext_tmem == kNoTmem) tmem_dealloc(tbase, TCOLS);
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
  // statistics of each (head, q head) row: reduce over the KPT keys of this head (the warp's
  // lanes; a 64-key head also merges its partner warp's half through shared memory)
  float lse[G];
#pragma unroll
  for (int g = 0; g < G; ++g) {
#pragma unroll
    for (int o = (KPT < 32 ? KPT : 32) / 2; o >= 1; o >>= 1) {
      const float om = __shfl_xor_sync(0xffffffffu, m[g], o), ol = __shfl_xor_sync(0xffffffffu, l[g], o);
      stat_merge(m[g], l[g], om, ol);
    }
  }
  if constexpr (KPT == 64) {
    float* xs = reinterpret_cast<float*>(smem + L.wm);  // [warp][G][m, l]
    if (lane == 0) {
#pragma unroll
      for (int g = 0; g < G; ++g) xs[(warp * G + g) * 2] = m[g], xs[(warp * G + g) * 2 + 1] = l[g];
    }
    sw_bar();
#pragma unroll
    for (int g = 0; g < G; ++g) stat_merge(m[g], l[g], xs[((warp ^ 1) * G + g) * 2], xs[((warp ^ 1) * G + g) * 2 + 1]);
  }
#pragma unroll
  for (int g = 0; g < G; ++g) lse[g] = m[g] + log2f(l[g]);
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

template <int G, int NR, int NSLOT, int TCOLS>
__global__ void __launch_bounds__(NT, TCOLS == 512 ? 1 : 2) attn_umma_kernel(const __grid_constant__ Params p) {
  verify_body<G, NR, NSLOT, TCOLS>(p, blockIdx.y, blockIdx.z);
}

// ---------------------------------------------------------------------------------------
// f3: one launch for a layer's verify AND draft work.  The grid is the verify launch (C-CTA
// clusters); a CTA that has finished its verify chunk (only once every verify CTA has
// started, unless any_cta) keeps claiming draft units ((item, group of four kv heads), the
// head-packed K1 body on the same six warps, one producer) from a global counter until none
// is left, so the draft work fills the verify launch's tail waves on chip instead of in a
// second launch.  Measured against the two launches on priority streams it loses (DESIGN.md
// §0 f3), so the layer loop uses it only with SD_ATTN_FUSED=1.
struct FusedCtl {
  unsigned int* ctr;  // [2 launch parities][next draft unit, verify CTAs started]: zero at the
                      // start of a launch (launch t clears parity t + 1 for the next launch on
                      // the stream), so plain atomicAdd, no reset launch
  int parity;         // this launch's counter pair
  int n_units;        // draft items x (kv heads / 4)
  int hgroups;        // kv heads / 4
  int n_ctas;         // verify CTAs of the launch
  int any_cta;        // 1: every CTA takes draft units after its verify chunk; 0: only those
                      // finishing once every verify CTA has started (the last wave)
};

template <int G, int NR, int NSLOT, int TCOLS>
__global__ void __launch_bounds__(NT, 2) attn_fused_kernel(const __grid_constant__ Params pv,
                                                           const __grid_constant__ Params pd, const FusedCtl fc) {
  // one TMEM allocation (256 columns) for both bodies
  __shared__ uint32_t s_tmem;
  __shared__ int s_unit;
  unsigned int* my = fc.ctr + 2 * fc.parity;
  if ((threadIdx.x >> 5) == WMMA) tmem_alloc(&s_tmem, TCOLS);
  if (threadIdx.x == 0) {
    atomicAdd(my + 1, 1u);  // this verify CTA has started
    if (blockIdx.x == 0 && blockIdx.y == 0 && blockIdx.z == 0) {  // the next launch's pair
      fc.ctr[2 * (fc.parity ^ 1)] = 0;
      fc.ctr[2 * (fc.parity ^ 1) + 1] = 0;
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tm = s_tmem;
  verify_body<G, NR, NSLOT, TCOLS>(pv, blockIdx.y, blockIdx.z, tm);
  // only CTAs finishing once every verify CTA has started take draft units: earlier ones
  // leave their cluster's slots to the verify clusters still waiting (no fragmentation),
  // the last wave's CTAs fill its tail with the drafts
  if (threadIdx.x == 0)
    s_unit = fc.any_cta || *reinterpret_cast<volatile unsigned int*>(my + 1) >= (unsigned)fc.n_ctas ? 0 : -1;
  __syncthreads();
  if (s_unit >= 0) {
    __syncthreads();
    for (;;) {
      if (threadIdx.x == 0) s_unit = (int)atomicAdd(my, 1u);
      __syncthreads();
      const int u = s_unit;
      __syncthreads();
      if (u >= fc.n_units) break;
      draft_body<G, 4, 2, 256, 1>(pd, u % fc.hgroups, u / fc.hgroups, tm);
      __syncthreads();
    }
  }
  tc_fence_before();
  __syncthreads();
  if ((threadIdx.x >> 5) == WMMA) {
    tc_fence_after();
    tmem_dealloc(tm, TCOLS);
  }
}

template <int G, int NR, int NSLOT, int TCOLS>
int launch_fused(const Params& pv, const Params& pd, const FusedCtl& fc, int C, int num_items, int kv_heads, int smem,
                 cudaStream_t stream) {
  auto kern = attn_fused_kernel<G, NR, NSLOT, TCOLS>;
  static int configured = 0;
  if (smem > configured) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
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
  cudaError_t e = cudaLaunchKernelEx(&cfg, kern, pv, pd, fc);
  count_launch();
  if (e != cudaSuccess) {
    set_error(std::string("sd_attention_pair (fused) launch: ") + cudaGetErrorString(e));
    return (int)e;
  }
  return 0;
}

// dynamic shared memory / cluster attributes of one instantiation (raised on demand)
template <int G, int NR, int NSLOT, int TCOLS>
void configure_verify(int smem) {
  static int configured = 0;
  if (smem > configured) {
    auto kern = attn_umma_kernel<G, NR, NSLOT, TCOLS>;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    configured = smem;
  }
}

// CTA slots the GPU offers C-CTA clusters of this instantiation at once: clusters live
// inside one GPC, so for C that do not divide a GPC's CTA slots this is well below
// 148 x CTAs-per-SM (the planner's wave count uses it)
template <int G, int NR, int NSLOT, int TCOLS>
int verify_slots(int C, int smem) {
  configure_verify<G, NR, NSLOT, TCOLS>(smem);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(C, 1, 1);
  cfg.blockDim = dim3(NT);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = C;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  int clusters = 0;
  if (cudaOccupancyMaxActiveClusters(&clusters, attn_umma_kernel<G, NR, NSLOT, TCOLS>, &cfg) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return clusters * C;
}

// launch one verify grid (C-CTA clusters) of attn_umma_kernel<G, NR, NSLOT, TCOLS>
template <int G, int NR, int NSLOT, int TCOLS>
int launch_verify(const Params& prm, int C, int num_items, int kv_heads, cudaStream_t stream) {
  constexpr int S = TCOLS / NR;
  auto kern = attn_umma_kernel<G, NR, NSLOT, TCOLS>;
  const int smem = make_layout(NR, NSLOT, S, prm.chunk / TK, prm.dense).total;
  configure_verify<G, NR, NSLOT, TCOLS>(smem);
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
    set_error(std::string("sd_attention (umma) launch: ") + cudaGetErrorString(e));
    return (int)e;
  }
  return 0;
}

// narrow = two CTAs per SM (256 TMEM columns, 2-slot ring); wide = one CTA per SM (512
// columns, 4-slot ring) for NR > 48, where m/l of every row no longer fit two CTAs' registers
constexpr int kNarrowMaxNR = 48;
constexpr int kMaxNR = 80;
int launch_verify_g4(const Params& prm, int NR, int C, int num_items, int kv_heads, cudaStream_t stream);
int launch_verify_g8(const Params& prm, int NR, int C, int num_items, int kv_heads, cudaStream_t stream);
// fused verify + draft launch for the two-CTA-per-SM verify shapes (NR <= 48); -1: no such
int launch_fused_g4(const Params& pv, const Params& pd, const FusedCtl& fc, int NR, int C, int num_items, int kv_heads,
                    int smem, cudaStream_t stream);
int launch_fused_g8(const Params& pv, const Params& pd, const FusedCtl& fc, int NR, int C, int num_items, int kv_heads,
                    int smem, cudaStream_t stream);
int verify_slots_g4(int NR, int C, int smem);

int verify_slots_g8(int NR, int C, int smem);

}  // namespace umma_attn
}  // namespace sd
