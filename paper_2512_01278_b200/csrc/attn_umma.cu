// tcgen05 (UMMA) paged attention for sm_100a: K2 verify with PillarAttn score
// emission and K1 sparse draft, every K and V row read from HBM exactly once.
//
// Orientation ("swap AB"): the KEYS of a 128-key tile are the UMMA M dimension
// and the item's query rows (token x GQA group, padded to NR) are N:
//
//   S^T[128 keys][NR] = K_tile[128][d] . Q^T            (kind::f16, K = d)
//   O^T[d][NR]       += V_tile^T[d][128] . P^T[128][NR]  (A MN-major, K = keys)
//
// so TMEM lane = key (phase 1/2) and lane = head-dim column (epilogue): each
// softmax thread owns ONE key and holds all NR query-row logits of it in
// registers.  Consequences:
//   * per-row online (max, sum) is thread-local across tiles; the cross-key
//     reduction happens once per CTA (shuffles + smem + DSMEM across the
//     cluster), not once per tile;
//   * the PillarAttn score  acc[token][pos] += sum_g exp(s - lse)  is a
//     register-local sum over the G group columns: one RED per (key, token);
//   * the planted bonus and the causal mask are per-key scalars.
//
// The logits of the CTA's whole key chunk stay in TMEM between the passes
// (up to TMAX tiles of NR fp32 columns), so the exact lse is known before
// any probability is formed (SURVEY.md §7.2 option (c)) without re-reading K.
//
//   grid = (C, kv_heads, items), cluster (C,1,1): CTA c owns keys
//   [c*chunk, (c+1)*chunk) of the item's key list (critical list, then the
//   dense causal range).
//   warps 0-3  softmax / scores / P^T -> smem / epilogue (TMEM lanes 0..127)
//   warp 4     producer: 16-byte cp.async of 256-byte key rows (paged gather)
//              into an NSLOT x 32 KB ring in the UMMA SWIZZLE_128B layout;
//              K tiles of the chunk, then V tiles (each row once)
//   warp 5     TMEM allocator + single-thread tcgen05.mma issuer
//
// Restates model.py:229-253 (_attend) for forward_full (model.py:318-334) and
// forward_sparse (model.py:360-380), and the score path selection.py:78-135.
#include "umma_common.cuh"

namespace sd {
namespace umma_attn {

template <int G, int NR, int NSLOT, int TCOLS>
__device__ __forceinline__ void verify_body(const Params& p, const int h, const int item_idx) {
  constexpr int TMAX = (TCOLS - NR) / NR;  // S tiles resident in TMEM (slot ring)
  constexpr int OCOL = TMAX * NR;          // O^T accumulator columns
  constexpr int NTOK = NR / G;             // token slots covered by NR rows

  cg::cluster_group cluster = cg::this_cluster();
  const int C = static_cast<int>(cluster.num_blocks());
  const int crank = static_cast<int>(cluster.block_rank());
  const Item it = load_item(p.items, item_idx);
  const int R = it.nq * G;
  const int Nk = it.num_keys();
  const int kb = crank * p.chunk;
  const int ke = min(Nk, kb + p.chunk);
  const int nk = max(0, ke - kb);
  const int nt = (nk + TK - 1) / TK;
  const int TR = min(nt, TMAX);
  const int nfill = 3 * nt - TR;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int cta_lin = (blockIdx.z * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x;
#define TRACE(k, val)                                                                                   \
  do {                                                                                                  \
    if (p.trace && cta_lin < kTraceCtas) g_trace[cta_lin * kTraceSlots + (k)] = (val);                  \
  } while (0)
  if (tid == 0) {
    uint32_t smid;
    asm volatile("mov.u32 %0, %smid;" : "=r"(smid));
    TRACE(0, gtime());
    TRACE(9, (uint64_t)smid | ((uint64_t)nt << 32));
  }

  extern __shared__ unsigned char smem_raw[];
  unsigned char* smem = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const Layout L = make_layout(NR, NSLOT, TMAX, p.chunk / TK, p.dense);
  unsigned char* ring = smem + L.ring;
  unsigned char* qs = smem + L.q;
  unsigned char* pbuf = smem + L.pbuf;
  int32_t* spos = reinterpret_cast<int32_t*>(smem + L.pos);
  int32_t* sslot = reinterpret_cast<int32_t*>(smem + L.slot);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + L.bar);
  uint64_t* empty = full + NSLOT;
  uint64_t* sfull = empty + NSLOT;       // [TMAX] logits of the slot's current use are in TMEM
  uint64_t* sfree = sfull + TMAX;        // [TMAX] softmax warps are done reading the slot
  uint64_t* pready = sfree + TMAX;       // [2] P^T buffer written
  uint64_t* pfree = pready + 2;          // [2] P^T buffer consumed by the PV MMA
  uint64_t* obar = pfree + 2;            // O^T complete
  float* wm = reinterpret_cast<float*>(smem + L.wm);
  float* wl = reinterpret_cast<float*>(smem + L.wl);
  float* xm = reinterpret_cast<float*>(smem + L.xm);
  float* xl = reinterpret_cast<float*>(smem + L.xl);
  float* rowlse = reinterpret_cast<float*>(smem + L.rowlse);
  uint32_t* tptr = reinterpret_cast<uint32_t*>(smem + L.tptr);

  // ---- setup ----
  if (warp == WMMA) tmem_alloc(tptr, TCOLS);
  if (tid == 0) {
    for (int i = 0; i < NSLOT; ++i) mbar_init(full + i, 32), mbar_init(empty + i, 1);
    for (int i = 0; i < TMAX; ++i) mbar_init(sfull + i, 1), mbar_init(sfree + i, NSW);
    mbar_init(pready + 0, NSW), mbar_init(pready + 1, NSW);
    mbar_init(pfree + 0, 1), mbar_init(pfree + 1, 1);
    mbar_init(obar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  // key positions and their physical slots for the whole chunk (the producer's copy loop
  // then never waits on a block-table load); keys past the chunk copy the last valid row
  // (finite data, masked out of the softmax).  Dense items stage only the page ids.
  const int32_t* trow = p.kv.table + (int64_t)it.table_row * p.kv.table_stride;
  const int pshift = p.kv.page_shift, pmask = (1 << pshift) - 1;
  const int dpos0 = it.dense_lo + kb;          // dense: position of chunk key 0
  const int dpage0 = dpos0 >> pshift;
  int32_t* spage = spos;                       // dense: [page - dpage0] -> physical page
  if (p.dense) {
    if (nk > 0) {
      const int lastpg = (it.dense_lo + ke - 1) >> pshift;
      const int npg = ((dpos0 + nt * TK - 1) >> pshift) - dpage0 + 1;
      for (int i = tid; i < npg; i += NT) spage[i] = __ldg(trow + min(dpage0 + i, lastpg));
    }
  } else {
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
  // Q rows (token-major: r = tok*G + g) -> [dhalf][NR][128 B] SWIZZLE_128B, zero padding rows
  for (int i = tid; i < NR * 16; i += NT) {
    const int r = i >> 4, c = i & 15;
    uint4 v = make_uint4(0, 0, 0, 0);
    if (r < R)
      v = *reinterpret_cast<const uint4*>(p.q + ((int64_t)(it.q_row0 + r / G) * p.q_heads + h * G + r % G) * D +
                                          c * 8);
    *reinterpret_cast<uint4*>(qs + (c >> 3) * (NR * 128) + r * 128 + (((c & 7) ^ (r & 7)) << 4)) = v;
  }
  fence_proxy_async();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = *tptr;
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
    for (int f = 0; f < nfill; ++f) {
      const int s = f % NSLOT;
      int t;
      bool isv;
      fill_tile(f, nt, TR, t, isv);
      const __nv_bfloat16* base = (isv ? Vg : Kg) + c * 8;
      int sl[4];  // physical slots of keys lane + 32m, broadcast by shuffles below
#pragma unroll
      for (int m = 0; m < 4; ++m) sl[m] = slot_of(t * TK + m * 32 + lane);
      if (f >= NSLOT) mbar_wait(empty + s, ((f / NSLOT) - 1) & 1);
      const uint32_t dst0 = ring_u + s * TILE_BYTES + (c >> 3) * (TK * 128);
#pragma unroll
      for (int kk = 0; kk < TK / 2; ++kk) {
        const int i = 2 * kk + sub;  // key row within the tile
        const int slot = __shfl_sync(0xffffffffu, sl[kk >> 4], i & 31);
        cp_async16(dst0 + i * 128 + (((c & 7) ^ (i & 7)) << 4), base + (int64_t)slot * row_stride, pol);
      }
      cp_async_mbar_arrive(full + s);
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
    // S^T for use u (tile's logits) into TMEM slot u % TMAX from ring slot s
    auto qk = [&](int u, int s) {
      mbar_wait(full + s, (f / NSLOT) & 1);
      if (u >= TMAX) mbar_wait(sfree + u % TMAX, ((u / TMAX) - 1) & 1);
      fence_proxy_async();
      tc_fence_after();
      if (leader) {
        const uint32_t a0 = ring_u + s * TILE_BYTES;
#pragma unroll
        for (int ks = 0; ks < D / 16; ++ks) {
          const uint32_t off = (ks & 3) << 5;  // K = 16 bf16 = 32 B steps inside the 128-B atom
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
    if (lane == 0) TRACE(10, gtime());
    if (C > 1) {
      cluster_wait();    // barrier 0
      cluster_arrive();  // barrier 1: this warp's part of phase 1 is issued
    }
    for (int i2 = 0; i2 < nt; ++i2) {
      if (i2 >= TR) qk(nt + (i2 - TR), f % NSLOT);  // evicted tile: recompute its logits
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
    tmem_dealloc(tbase, TCOLS);
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
  auto release = [&](int u) {  // one elected arrival per warp
    tc_fence_before();
    __syncwarp();
    if (lane == 0) mbar_arrive(sfree + u % TMAX);
  };

  // ---- phase 1: S^T tiles -> thread-local online (max, sum) ----
  for (int t = 0; t < nt; ++t) {
    int pos, rmin;
    float bias;
    key_info(t, pos, bias, rmin);
    mbar_wait(sfull + t % TMAX, (t / TMAX) & 1);
    tc_fence_after();
    float v[NR];
    tmem_ld_row<NR>(tl + (t % TMAX) * NR, v);
    if (t < nt - TR) release(t);  // evicted before phase 2: recomputed there
#pragma unroll
    for (int r = 0; r < NR; ++r) {
      if (r >= rmin && r < R) {
        const float s2 = fmaf(v[r], p.scale_log2, bias);
        const float nm = fmaxf(m[r], s2);
        l[r] = l[r] * ex2(m[r] - nm) + ex2(s2 - nm);
        m[r] = nm;
      }
    }
  }
  if (tid == 0) TRACE(2, gtime());
  // ---- exchange: warp -> CTA -> cluster row statistics -> exact lse ----
#pragma unroll
  for (int b0 = 0; b0 < NR; b0 += 32) {
    constexpr int NB0 = NR < 32 ? NR : 32;
    if (NR - b0 >= 32 || NR < 32) {
      warp_rows_reduce<NB0>(m + b0, l + b0, lane);
      const int row = b0 + (lane & (NB0 - 1));
      if (lane < NB0 && row < R) wm[warp * NR + row] = m[b0], wl[warp * NR + row] = l[b0];
    } else {  // NR = 48: rows 32..47
      warp_rows_reduce<16>(m + b0, l + b0, lane);
      const int row = b0 + (lane & 15);
      if (lane < 16 && row < R) wm[warp * NR + row] = m[b0], wl[warp * NR + row] = l[b0];
    }
  }
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
  float lse[NR];
#pragma unroll
  for (int r = 0; r < NR; ++r) lse[r] = rowlse[r];
  if (tid == 0) TRACE(3, gtime());

  // ---- phase 2: P = exp2(S - lse) (final), scores, P^T -> smem for the PV MMA ----
  const bool scores = p.acc != nullptr && it.acc_row >= 0;
  for (int i2 = 0; i2 < nt; ++i2) {
    const int t = i2 < TR ? nt - TR + i2 : i2 - TR;  // resident tiles first, then the evicted ones
    const int u = i2 < TR ? t : nt + t;              // TMEM slot use holding its logits
    int pos, rmin;
    float bias;
    key_info(t, pos, bias, rmin);
    mbar_wait(sfull + u % TMAX, (u / TMAX) & 1);
    tc_fence_after();
    float v[NR];
    tmem_ld_row<NR>(tl + (u % TMAX) * NR, v);
    release(u);
#pragma unroll
    for (int r = 0; r < NR; ++r)
      v[r] = (r >= rmin && r < R) ? ex2(fmaf(v[r], p.scale_log2, bias) - lse[r]) : 0.f;
    if (scores && rmin < R) {
      if (it.acc_step == 0) {
        float sum = 0.f;
#pragma unroll
        for (int r = 0; r < NR; ++r) sum += v[r];
        if (sum != 0.f) red_add(p.acc + (int64_t)it.acc_row * p.acc_stride + pos, sum);
      } else {
#pragma unroll
        for (int tk = 0; tk < NTOK; ++tk) {
          float sum = 0.f;
#pragma unroll
          for (int g = 0; g < G; ++g) sum += v[tk * G + g];
          if (sum != 0.f)
            red_add(p.acc + (int64_t)(it.acc_row + tk * it.acc_step) * p.acc_stride + pos, sum);
        }
      }
    }
    if (i2 >= 2) mbar_wait(pfree + (i2 & 1), ((i2 >> 1) - 1) & 1);
    // P^T [key][row]: core matrix (8 keys x 8 rows) = 128 B; key groups 128 B apart,
    // row groups TK*16 B apart -> this thread's 8-row chunks at kl*16 + ng*TK*16
    unsigned char* pb = pbuf + (i2 & 1) * (NR * TK * 2) + kl * 16;
#pragma unroll
    for (int ng = 0; ng < NR / 8; ++ng) {
      __nv_bfloat162 b0 = __floats2bfloat162_rn(v[ng * 8 + 0], v[ng * 8 + 1]);
      __nv_bfloat162 b1 = __floats2bfloat162_rn(v[ng * 8 + 2], v[ng * 8 + 3]);
      __nv_bfloat162 b2 = __floats2bfloat162_rn(v[ng * 8 + 4], v[ng * 8 + 5]);
      __nv_bfloat162 b3 = __floats2bfloat162_rn(v[ng * 8 + 6], v[ng * 8 + 7]);
      uint4 w;
      w.x = *reinterpret_cast<uint32_t*>(&b0);
      w.y = *reinterpret_cast<uint32_t*>(&b1);
      w.z = *reinterpret_cast<uint32_t*>(&b2);
      w.w = *reinterpret_cast<uint32_t*>(&b3);
      *reinterpret_cast<uint4*>(pb + ng * TK * 16) = w;
    }
    fence_proxy_async();
    __syncwarp();
    if (lane == 0) mbar_arrive(pready + (i2 & 1));
  }

  // ---- epilogue: O^T (lane = d) -> cluster reduction -> out ----
  if (tid == 0) TRACE(4, gtime());
  float o[NR];
  if (nt > 0) {
    mbar_wait(obar, 0);
    tc_fence_after();
    if (tid == 0) TRACE(5, gtime());
    tmem_ld_row<NR>(tl + OCOL, o);
  } else {
#pragma unroll
    for (int r = 0; r < NR; ++r) o[r] = 0.f;
  }
  tc_fence_before();
  asm volatile("bar.arrive 2, %0;\n" ::"n"((NSW + 1) * 32) : "memory");  // O read: TMEM may be freed
  const int dcol = kl;
  if (C == 1) {
#pragma unroll
    for (int r = 0; r < NR; ++r)
      if (r < R)
        p.out[((int64_t)(it.q_row0 + r / G) * p.q_heads + h * G + r % G) * D + dcol] = __float2bfloat16_rn(o[r]);
  } else {
    // all MMAs of this CTA are complete (obar): its ring holds the O^T partial; row r is
    // summed over the cluster by CTA r % C (DSMEM loads issued back to back)
    float* Ob = reinterpret_cast<float*>(ring);  // [NR][D]
#pragma unroll
    for (int r = 0; r < NR; ++r)
      if (r < R) Ob[r * D + dcol] = o[r];
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

template <int G, int NR, int NSLOT, int TCOLS>
__global__ void __launch_bounds__(NT, TCOLS == 512 ? 1 : 2) attn_umma_kernel(const Params p) {
  verify_body<G, NR, NSLOT, TCOLS>(p, blockIdx.y, blockIdx.z);
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

  if (warp == WMMA) tmem_alloc(tptr, TCOLS);
  if (tid == 0) {
    for (int i = 0; i < NSLOT; ++i) mbar_init(full + i, 32), mbar_init(empty + i, 1);
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
    for (int j0 = 0; j0 < nkeys; j0 += 8 * NT) {
      int pos[8], pg[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) pos[k] = it.key_pos(p.crit, min(j0 + k * NT + tid, nk - 1));
#pragma unroll
      for (int k = 0; k < 8; ++k) pg[k] = __ldg(trow + (pos[k] >> p.kv.page_shift));
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const int j = j0 + k * NT + tid;
        if (j < nkeys) {
          spos[j] = j < nk ? pos[k] : -1;
          sslot[j] = (pg[k] << p.kv.page_shift) | (pos[k] & pmask);
        }
      }
    }
  }
  // Q: the CTA's NQ q heads are contiguous in the row (heads h0.. x group)
  for (int i = tid; i < NR * 16; i += NT) {
    const int r = i >> 4, c = i & 15;
    uint4 v = make_uint4(0, 0, 0, 0);
    if (r < NQ) v = *reinterpret_cast<const uint4*>(p.q + ((int64_t)it.q_row0 * p.q_heads + h0 * G + r) * D + c * 8);
    *reinterpret_cast<uint4*>(qs + (c >> 3) * (NR * 128) + r * 128 + (((c & 7) ^ (r & 7)) << 4)) = v;
  }
  // P^T buffers: off-diagonal blocks stay zero for the whole launch
  for (int i = tid; i < 2 * NR * TK * 2 / 16; i += NT) reinterpret_cast<uint4*>(pbuf)[i] = make_uint4(0, 0, 0, 0);
  fence_proxy_async();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = *tptr;

  const int64_t row_stride = (int64_t)p.kv.kv_heads * D;
  const __nv_bfloat16* Kg = static_cast<const __nv_bfloat16*>(p.kv.k) + (int64_t)p.layer * p.kv.layer_stride + h0 * D;
  const __nv_bfloat16* Vg = static_cast<const __nv_bfloat16*>(p.kv.v) + (int64_t)p.layer * p.kv.layer_stride + h0 * D;

  if (warp == WPROD) {
    const uint64_t pol = policy_evict_first();
    const int sub = lane >> 4, c = lane & 15;
    const uint32_t ring_u = smem_u32(ring);
    for (int f = 0; f < nfill; ++f) {
      const int s = f % NSLOT;
      int t;
      bool isv;
      fill_tile(f, nt, TR, t, isv);
      const __nv_bfloat16* base = (isv ? Vg : Kg) + c * 8;
      const int sl = sslot[t * KPT + (lane % KPT)];
      if (f >= NSLOT) mbar_wait(empty + s, ((f / NSLOT) - 1) & 1);
      const uint32_t dst0 = ring_u + s * TILE_BYTES + (c >> 3) * (TK * 128);
#pragma unroll
      for (int kk = 0; kk < TK / 2; ++kk) {
        const int i = 2 * kk + sub;            // tile row = head-major (hh, key)
        const int hh = (2 * kk) / KPT;         // same for both rows of the instruction
        const int slot = __shfl_sync(0xffffffffu, sl, ((2 * kk) % KPT) + sub);
        cp_async16(dst0 + i * 128 + (((c & 7) ^ (i & 7)) << 4), base + (int64_t)slot * row_stride + hh * D, pol);
      }
      cp_async_mbar_arrive(full + s);
    }
    return;
  }

  if (warp == WMMA) {
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
    if (scores && sum != 0.f) red_add(p.acc + (int64_t)it.acc_row * p.acc_stride + pos, sum);
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
  if (nt > 0) {
    mbar_wait(obar, 0);
    tc_fence_after();
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
}

template <int G, int HPC, int NSLOT, int TCOLS>
__global__ void __launch_bounds__(NT, TCOLS == 512 ? 1 : 2) attn_umma_hp_kernel(const Params p) {
  draft_body<G, HPC, NSLOT, TCOLS>(p, blockIdx.x, blockIdx.y);
}

// f3: one launch for a layer's verify (K2) and draft (K1) work.  The grid holds the verify
// clusters first (blockIdx.z < nv: unit z = item z / Hkv, head z % Hkv, chunk = cluster
// rank) and then clusters of C head-packed draft CTAs (no cluster cooperation among them),
// so the block scheduler fills the verify launch's tail wave with draft work instead of
// running the drafts as a separate, under-filled launch.
template <int G, int NRV, int NSLOT, int TCOLS>
__global__ void __launch_bounds__(NT, 2) attn_fused_kernel(const Params pv, const Params pd, int nv, int nd) {
  const int z = blockIdx.z;
  if (z < nv) {
    verify_body<G, NRV, NSLOT, TCOLS>(pv, z % pv.kv.kv_heads, z / pv.kv.kv_heads);
    return;
  }
  const int dc = (z - nv) * gridDim.x + blockIdx.x;
  if (dc >= nd) return;
  const int groups = pd.kv.kv_heads / 4;
  draft_body<G, 4, NSLOT, TCOLS>(pd, dc % groups, dc / groups);
}

template <int G, int HPC, int NSLOT, int TCOLS>
int launch_hp(const Params& prm, int num_items, int kv_heads, int ct, cudaStream_t stream) {
  constexpr int NQ = HPC * G, NR = NQ < 16 ? 16 : NQ, TMAX = (TCOLS - NR) / NR;
  auto kern = attn_umma_hp_kernel<G, HPC, NSLOT, TCOLS>;
  const int smem = make_hp_layout(NR, NSLOT, TMAX, ct).total;
  static int configured = 0;
  if (smem > configured) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    configured = smem;
  }
  kern<<<dim3(kv_heads / HPC, num_items), NT, smem, stream>>>(prm);
  count_launch();
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_error(std::string("sd_attention (umma, head-packed) launch: ") + cudaGetErrorString(e));
    return (int)e;
  }
  return 0;
}

template <int G, int NR, int NSLOT, int TCOLS>
int launch_one(const Params& prm, int C, int num_items, int kv_heads, cudaStream_t stream) {
  constexpr int TMAX = (TCOLS - NR) / NR;
  auto kern = attn_umma_kernel<G, NR, NSLOT, TCOLS>;
  const int smem = make_layout(NR, NSLOT, TMAX, prm.chunk / TK, prm.dense).total;
  static int configured = 0;
  if (smem > configured) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, 100);  // two CTAs per SM
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
    set_error(std::string("sd_attention (umma) launch: ") + cudaGetErrorString(e));
    return (int)e;
  }
  return 0;
}

static int env_int(const char* name, int dflt) {
  const char* v = getenv(name);
  return v && *v ? atoi(v) : dflt;
}

// Key tiles of one CTA's chunk that fit the shared-memory budget (positions + slots staged per key).
static int chunk_cap_tiles(int NR, int nslot, int tmax, int budget, int dense) {
  int ct = 1;
  while (ct < 512 && make_layout(NR, nslot, tmax, ct + 1, dense).total <= budget) ++ct;
  return make_layout(NR, nslot, tmax, ct, dense).total <= budget ? ct : 0;
}

}  // namespace umma_attn

// Cluster size C (<= 16) and chunk for one launch: minimise (waves of SM slots) x
// (32 KB fills per CTA + fixed per-CTA cost ~7 fills, fitted to traced C sweeps).  Chunks longer than the TMEM-resident
// tiles re-read the evicted tiles' K in phase 2 (fills = 3*ct - tmax).
static bool plan_umma(int max_keys, int num_items, int kv_heads, int tmax, int cap, int slots, int* C_out,
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
    const double fills = ct <= tmax ? 2.0 * ct : 3.0 * ct - tmax;
    const long long ctas = work * c;
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

struct UmmaPlan {
  int NR, C, chunk;
  bool wide;
};

static bool umma_plan(const sd_paged_kv* kvp, int num_items, int max_keys, int max_nq, int q_heads, int dense,
                      UmmaPlan* pl) {
  using namespace umma_attn;
  const int G = q_heads / kvp->kv_heads;
  if (kvp->dtype != SD_DTYPE_BF16 || kvp->head_dim != D) return false;
  if (!(G == 4 || G == 8)) return false;
  const int rows = max_nq * G;
  const int NR = rows <= 16 ? 16 : rows <= 32 ? 32 : rows <= 48 ? 48 : rows <= 64 ? 64 : 0;
  if (NR == 0 || NR % G != 0) return false;
  static const int wide_env = env_int("SD_UMMA_WIDE", -1);  // 1: one CTA/SM, 512 TMEM columns, 5-slot ring
  // two CTAs per SM (256 TMEM columns, 2-slot ring each) unless their shared memory does not fit
  const int narrow_cap = chunk_cap_tiles(NR, 2, (256 - NR) / NR, 113 * 1024, dense);
  const int wide_cap = chunk_cap_tiles(NR, 5, (512 - NR) / NR, 227 * 1024, dense);
  const int mk = max_keys < 1 ? 1 : max_keys;
  int C = 1, chunk = TK;
  bool wide = false;
  if (!(wide_env != 1 && narrow_cap > 0 &&
        plan_umma(mk, num_items, kvp->kv_heads, (256 - NR) / NR, narrow_cap, 296, &C, &chunk, dense))) {
    if (wide_env == 0 || wide_cap == 0 ||
        !plan_umma(mk, num_items, kvp->kv_heads, (512 - NR) / NR, wide_cap, 148, &C, &chunk, dense))
      return false;
    wide = true;
  }
  pl->NR = NR, pl->C = C, pl->chunk = chunk, pl->wide = wide;
  return true;
}

int64_t umma_ws_bytes(const sd_paged_kv* kvp, int num_items, int max_keys, int max_nq, int q_heads, bool* handled) {
  UmmaPlan pl;
  *handled = umma_plan(kvp, num_items, max_keys, max_nq, q_heads, 1, &pl);
  return 0;  // O partials meet in DSMEM: no workspace
}

int launch_attn_umma(const void* q, void* out, float* lse, const sd_paged_kv* kvp, int layer, const int32_t* items,
                     int num_items, int max_keys, int max_nq, const int32_t* crit, float* acc, int64_t acc_stride,
                     const int32_t* planted, int n_planted, float bonus, int q_heads, float scale, void* ws,
                     int64_t ws_bytes, cudaStream_t stream, bool* handled) {
  using namespace umma_attn;
  *handled = false;
  static const int hp_env = env_int("SD_UMMA_HP", 1);
  {
    const int G = q_heads / kvp->kv_heads;
    if (hp_env && max_nq == 1 && kvp->dtype == SD_DTYPE_BF16 && kvp->head_dim == D && (G == 4 || G == 8) &&
        kvp->kv_heads % 4 == 0) {
      // 4 heads per CTA, 32 keys per tile, the whole key list in one CTA
      const int NR = 4 * G, tmax = (256 - NR) / NR;
      const int ct_tiles = (max(max_keys, 1) + 31) / 32;      // 32-key tiles
      const int ct = (ct_tiles * 32 + TK - 1) / TK;           // 128-key units for the staging arrays
      if (ct_tiles <= tmax && make_hp_layout(NR, 2, tmax, ct).total <= 113 * 1024) {  // logits stay resident
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
        prm.planted = planted;
        prm.n_planted = n_planted;
        prm.bonus_log2 = bonus * LOG2E;
        prm.q_heads = q_heads;
        prm.scale_log2 = scale * LOG2E;
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
  }
  UmmaPlan pl;
  const int dense = (crit == nullptr && kvp->page_shift >= 4) ? 1 : 0;
  if (!umma_plan(kvp, num_items, max_keys, max_nq, q_heads, dense, &pl)) return 0;
  const int G = q_heads / kvp->kv_heads;
  const int NR = pl.NR, C = pl.C;
  const bool wide = pl.wide;
  Params prm;
  (void)ws;
  (void)ws_bytes;
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
  prm.chunk = pl.chunk;
  prm.dense = dense;
  static const int trace = env_int("SD_ATTN_TRACE", 0);
  prm.trace = trace;
  *handled = true;
#define SD_UMMA_CASE(GG, N)                                                                   \
  if (G == GG && NR == N) {                                                                   \
    if (wide) return launch_one<GG, N, 5, 512>(prm, C, num_items, kvp->kv_heads, stream);     \
    return launch_one<GG, N, 2, 256>(prm, C, num_items, kvp->kv_heads, stream);               \
  }
  SD_UMMA_CASE(4, 16) SD_UMMA_CASE(4, 32) SD_UMMA_CASE(4, 48) SD_UMMA_CASE(4, 64)
  SD_UMMA_CASE(8, 16) SD_UMMA_CASE(8, 32) SD_UMMA_CASE(8, 48) SD_UMMA_CASE(8, 64)
#undef SD_UMMA_CASE
  *handled = false;
  return 0;
}

// f3 fused launch of one layer's verify launch (items_v, K2 with score capture) and draft
// launch (items_d, K1 over critical lists) when both fit the tcgen05 kernels; otherwise
// *handled = false and the caller issues the two launches separately.
int launch_attn_fused(const void* q, void* out, const sd_paged_kv* kvp, int layer, const int32_t* items_v,
                      int nv_items, int v_max_keys, int v_max_nq, float* acc, int64_t acc_stride,
                      const int32_t* items_d, int nd_items, int d_max_keys, const int32_t* crit,
                      const int32_t* planted, int n_planted, float bonus, int q_heads, float scale,
                      cudaStream_t stream, bool* handled) {
  using namespace umma_attn;
  *handled = false;
  // measured: device-only configs[1] forward 8.52 ms fused vs 8.30 ms as two launches (the
  // draft CTAs queue behind the verify clusters instead of filling their tail): off by default
  static const int enable = env_int("SD_ATTN_FUSED", 0);
  const int G = q_heads / kvp->kv_heads;
  if (!enable || nv_items == 0 || nd_items == 0 || v_max_nq < 2) return 0;
  if (kvp->dtype != SD_DTYPE_BF16 || kvp->head_dim != D || !(G == 4 || G == 8) || kvp->kv_heads % 4 != 0) return 0;
  UmmaPlan pl;
  const int dense = kvp->page_shift >= 4 ? 1 : 0;
  if (!umma_plan(kvp, nv_items, v_max_keys, v_max_nq, q_heads, dense, &pl) || pl.wide || pl.NR > 48) return 0;
  const int NRD = 4 * G, tmax_d = (256 - NRD) / NRD;
  const int ct_tiles = (max(d_max_keys, 1) + 31) / 32;
  const int ct_d = (ct_tiles * 32 + TK - 1) / TK;
  if (ct_tiles > tmax_d) return 0;
  const int tmax_v = (256 - pl.NR) / pl.NR;
  const int smem = max(make_layout(pl.NR, 2, tmax_v, pl.chunk / TK, dense).total, make_hp_layout(NRD, 2, tmax_d, ct_d).total);
  if (smem > 113 * 1024) return 0;
  static const int trace = env_int("SD_ATTN_TRACE", 0);
  if (trace) return 0;
  Params pv{}, pd{};
  for (Params* pp : {&pv, &pd}) {
    pp->q = static_cast<const __nv_bfloat16*>(q);
    pp->out = static_cast<__nv_bfloat16*>(out);
    pp->lse_out = nullptr;
    pp->kv = make_paged(kvp);
    pp->layer = layer;
    pp->planted = planted;
    pp->n_planted = n_planted;
    pp->bonus_log2 = bonus * LOG2E;
    pp->q_heads = q_heads;
    pp->scale_log2 = scale * LOG2E;
  }
  pv.items = items_v, pv.acc = acc, pv.acc_stride = acc_stride, pv.chunk = pl.chunk, pv.dense = dense;
  pd.items = items_d, pd.crit = crit, pd.chunk = ct_d * TK;
  const int C = pl.C;
  const int nv = nv_items * kvp->kv_heads;
  const int nd = nd_items * (kvp->kv_heads / 4);
  const int nz = nv + (nd + C - 1) / C;
  auto go = [&](auto kern) -> int {
    static int configured = 0;
    if (smem > configured) {
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
      cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
      configured = smem;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(C, 1, nz);
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
    cudaError_t e = cudaLaunchKernelEx(&cfg, kern, pv, pd, nv, nd);
    count_launch();
    if (e != cudaSuccess) {
      set_error(std::string("sd_attention (fused draft + verify) launch: ") + cudaGetErrorString(e));
      return (int)e;
    }
    return 0;
  };
  *handled = true;
  if (G == 4) {
    if (pl.NR == 16) return go(attn_fused_kernel<4, 16, 2, 256>);
    if (pl.NR == 32) return go(attn_fused_kernel<4, 32, 2, 256>);
    return go(attn_fused_kernel<4, 48, 2, 256>);
  }
  if (pl.NR == 32) return go(attn_fused_kernel<8, 32, 2, 256>);
  if (pl.NR == 48) return go(attn_fused_kernel<8, 48, 2, 256>);
  *handled = false;
  return 0;
}

}  // namespace sd

// Diagnostics: per-CTA phase timestamps of the last traced umma launch (SD_ATTN_TRACE=1):
// [ctas][10] uint64 = start, setup done, phase 1 done, lse known, phase 2 done, O ready,
// end, producer done, -, smid | tiles << 32.
extern "C" int sd_attention_trace_umma(uint64_t* host_dst, int32_t ctas) {
  if (ctas > sd::umma_attn::kTraceCtas) ctas = sd::umma_attn::kTraceCtas;
  cudaError_t e = cudaMemcpyFromSymbol(host_dst, sd::umma_attn::g_trace,
                                       sizeof(uint64_t) * sd::umma_attn::kTraceSlots * ctas);
  return e == cudaSuccess ? 0 : (int)e;
}
