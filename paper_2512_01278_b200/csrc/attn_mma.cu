// Tensor-core (bf16 mma.sync m16n8k16) paged attention for sm_100a with a
// thread-block cluster per (work item, kv head) and exact two-phase softmax.
//
//   grid    = (C, kv_heads, num_items), cluster = (C, 1, 1)
//   CTA c   = keys [c*chunk, (c+1)*chunk) of the item's key list
//             (critical positions first, then the dense causal range)
//
// phase 1  K tiles (64 keys) stream HBM -> smem with a 4-stage cp.async ring;
//          S^T tile = Q K^T on tensor cores; scaled/masked/planted logits are
//          kept in shared memory for the whole chunk (log2 domain).
// exchange per-row (max, sum) across the cluster through DSMEM -> exact lse.
// phase 2  V tiles stream in; P = exp2(S - lse) is FINAL (no online
//          rescaling), so PillarAttn's score accumulator
//          acc[token][pos] += sum_{g in group} P  is emitted right here, with
//          zero extra HBM traffic for logits (SURVEY.md §7.2 option (c));
//          O_partial = P V on tensor cores.
// reduce   O partials summed across the cluster through DSMEM, written once.
//
// Restates model.py:229-253 (_attend), used by forward_full (verify, prefill;
// model.py:318-334) and forward_sparse (draft; model.py:360-380), and the
// score path selection.py:78-135.
#include <cooperative_groups.h>

#include "common.cuh"

namespace cg = cooperative_groups;

namespace sd {
namespace mma_attn {

constexpr int TK = 64;      // keys per tile
constexpr int NT = 256;     // threads per CTA
constexpr int NW = NT / 32;
constexpr int STAGES = 4;
constexpr int PROW = TK + 8;  // bf16 per P-tile row (conflict-free ldmatrix)
constexpr float LOG2E = 1.4426950408889634f;
constexpr float LN2 = 0.6931471805599453f;

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, int src_bytes) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(src_bytes));
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
__device__ __forceinline__ void ldsm_x2_t(unsigned& r0, unsigned& r1, const void* p) {
  const unsigned a = static_cast<unsigned>(__cvta_generic_to_shared(p));
  asm volatile("ldmatrix.sync.aligned.m8n8.x2.trans.shared.b16 {%0,%1}, [%2];\n" : "=r"(r0), "=r"(r1) : "r"(a));
}
__device__ __forceinline__ void mma_bf16(float (&c)[4], unsigned a0, unsigned a1, unsigned a2, unsigned a3,
                                         unsigned b0, unsigned b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};\n"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
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
  int chunk;      // keys per CTA, multiple of TK
  int srow;       // floats per S row (chunk + 8)
  int s_rows;     // rows of the S buffer (max rows over items)
};

// Shared-memory carve, identical on host and device.
struct Layout {
  int k_off, q_off, p_off, s_off, pos_off, slot_off, m_off, l_off, lse_off, total;
};
__host__ __device__ inline Layout make_layout(int D, int MT, int chunk, int s_rows) {
  const int RP = MT * 16;
  const int krow = D + 8;
  Layout L;
  int o = 0;
  L.k_off = o;   o += STAGES * TK * krow * 2;
  L.q_off = o;   o += RP * krow * 2;
  L.p_off = o;   o += RP * PROW * 2;
  L.s_off = o;
  {
    const int s_bytes = s_rows * (chunk + 8) * 4;
    const int o_bytes = RP * D * 4;
    o += s_bytes > o_bytes ? s_bytes : o_bytes;
  }
  L.pos_off = o;  o += chunk * 4;
  L.slot_off = o; o += chunk * 4;
  L.m_off = o;    o += RP * 4;
  L.l_off = o;    o += RP * 4;
  L.lse_off = o;  o += RP * 4;
  L.total = o;
  return L;
}

template <int D, int MT>
__global__ void __launch_bounds__(NT, 1) attn_mma_kernel(const Params p) {
  constexpr int RP = MT * 16;
  constexpr int KROW = D + 8;
  constexpr int DCH = D / 8;          // 16-byte chunks per key row
  constexpr int NCOLW = D / NW;       // output columns per warp in phase 2 (16 or 8)
  constexpr int NTW = NCOLW / 8;      // n8 tiles per warp in phase 2

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
  const Layout L = make_layout(D, MT, p.chunk, p.s_rows);
  __nv_bfloat16* Kst = reinterpret_cast<__nv_bfloat16*>(smem + L.k_off);
  __nv_bfloat16* Qs = reinterpret_cast<__nv_bfloat16*>(smem + L.q_off);
  __nv_bfloat16* Pt = reinterpret_cast<__nv_bfloat16*>(smem + L.p_off);
  float* Sb = reinterpret_cast<float*>(smem + L.s_off);
  int32_t* spos = reinterpret_cast<int32_t*>(smem + L.pos_off);
  int32_t* sslot = reinterpret_cast<int32_t*>(smem + L.slot_off);
  float* rowm = reinterpret_cast<float*>(smem + L.m_off);
  float* rowl = reinterpret_cast<float*>(smem + L.l_off);
  float* rowlse = reinterpret_cast<float*>(smem + L.lse_off);

  const __nv_bfloat16* Kg = static_cast<const __nv_bfloat16*>(p.kv.k) + (int64_t)p.layer * p.kv.layer_stride;
  const __nv_bfloat16* Vg = static_cast<const __nv_bfloat16*>(p.kv.v) + (int64_t)p.layer * p.kv.layer_stride;
  const int kvh = p.kv.kv_heads;

  // ---- keys of this chunk: absolute position and physical slot ----
  for (int j = tid; j < ntiles * TK; j += NT) {
    const int gj = kb + j;
    if (gj < ke) {
      const int pos = it.key_pos(p.crit, gj);
      spos[j] = pos;
      sslot[j] = static_cast<int32_t>(p.kv.slot_of(it.table_row, pos));
    } else {
      spos[j] = 0x7fffffff;
      sslot[j] = -1;
    }
  }
  // ---- query rows (r = token * G + g), zero padded to RP ----
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

  auto load_tile = [&](const __nv_bfloat16* base, int t, int stage) {
#pragma unroll
    for (int i = tid; i < TK * DCH; i += NT) {
      const int kk = i / DCH, c = i - kk * DCH;
      const int slot = sslot[t * TK + kk];
      const __nv_bfloat16* src = base + ((int64_t)(slot < 0 ? 0 : slot) * kvh + h) * D + c * 8;
      cp_async16(Kst + (stage * TK + kk) * KROW + c * 8, src, slot < 0 ? 0 : 16);
    }
  };

  // ================= phase 1: logits =================
#pragma unroll
  for (int s = 0; s < STAGES - 1; ++s) {
    if (s < ntiles) load_tile(Kg, s, s);
    cp_async_commit();
  }
  for (int t = 0; t < ntiles; ++t) {
    cp_async_wait<STAGES - 2>();
    __syncthreads();
    {
      const int nt = t + STAGES - 1;
      if (nt < ntiles) load_tile(Kg, nt, nt % STAGES);
      cp_async_commit();
    }
    const __nv_bfloat16* Kt = Kst + (t % STAGES) * TK * KROW;
    float sacc[MT][4];
#pragma unroll
    for (int mt = 0; mt < MT; ++mt) sacc[mt][0] = sacc[mt][1] = sacc[mt][2] = sacc[mt][3] = 0.f;
    const int n0 = warp * 8;  // this warp's 8 keys of the tile
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
        mma_bf16(sacc[mt], a0, a1, a2, a3, b2, b3);
      }
    }
    // epilogue: scale, causal/extent mask, planted bonus -> S buffer (log2 domain)
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const int jl = t * TK + n0 + 2 * t4 + e;  // local key index
      const int gj = kb + jl;
      const int pos = spos[jl];
      const bool in_range = gj < ke;
      const bool is_crit = gj < it.crit_len;
      const float bias = in_range ? planted_bias(p.planted, p.n_planted, p.bonus_log2, pos) : 0.f;
#pragma unroll
      for (int mt = 0; mt < MT; ++mt) {
#pragma unroll
        for (int hh = 0; hh < 2; ++hh) {
          const int r = mt * 16 + g4 + hh * 8;
          if (r < R) {
            const bool vis = in_range && (is_crit || pos <= it.qpos0 + r / G);
            Sb[r * p.srow + jl] = vis ? fmaf(sacc[mt][hh * 2 + e], p.scale_log2, bias) : -INFINITY;
          }
        }
      }
    }
  }
  cp_async_wait<0>();
  __syncthreads();

  // prefetch the first V tiles while the softmax statistics are exchanged
#pragma unroll
  for (int s = 0; s < STAGES - 1; ++s) {
    if (s < ntiles) load_tile(Vg, s, s);
    cp_async_commit();
  }

  // ---- per-row chunk statistics ----
  for (int r = warp; r < RP; r += NW) {
    float m = -INFINITY, l = 0.f;
    if (r < R) {
      const float* Sr = Sb + r * p.srow;
      for (int j = lane; j < nk; j += 32) m = fmaxf(m, Sr[j]);
      m = warp_max(m);
      if (m != -INFINITY)
        for (int j = lane; j < nk; j += 32) l += exp2f(Sr[j] - m);
      l = warp_sum(l);
    }
    if (lane == 0) {
      rowm[r] = m;
      rowl[r] = l;
    }
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
  // zero the P-tile padding rows once
  for (int i = tid; i < (RP - R) * PROW; i += NT) Pt[R * PROW + i] = __float2bfloat16_rn(0.f);
  __syncthreads();

  // ================= phase 2: P, scores, O = P V =================
  const bool scores = p.acc != nullptr && it.acc_row >= 0;
  float oacc[MT][NTW][4];
#pragma unroll
  for (int mt = 0; mt < MT; ++mt)
#pragma unroll
    for (int nt = 0; nt < NTW; ++nt) oacc[mt][nt][0] = oacc[mt][nt][1] = oacc[mt][nt][2] = oacc[mt][nt][3] = 0.f;

  for (int t = 0; t < ntiles; ++t) {
    cp_async_wait<STAGES - 2>();
    __syncthreads();
    {
      const int nt = t + STAGES - 1;
      if (nt < ntiles) load_tile(Vg, nt, nt % STAGES);
      cp_async_commit();
    }
    // P tile (bf16) + score emission; thread -> (key, token lane)
    {
      const int kk = tid & (TK - 1);
      const int jl = t * TK + kk;
      const bool valid = (kb + jl) < ke;
      for (int qt = tid / TK; qt < it.nq; qt += NT / TK) {
        float sum = 0.f;
        for (int g = 0; g < G; ++g) {
          const int r = qt * G + g;
          const float pv = valid ? exp2f(Sb[r * p.srow + jl] - rowlse[r]) : 0.f;
          Pt[r * PROW + kk] = __float2bfloat16_rn(pv);
          sum += pv;
        }
        if (scores && sum != 0.f)
          atomicAdd(p.acc + (int64_t)(it.acc_row + qt * it.acc_step) * p.acc_stride + spos[jl], sum);
      }
    }
    __syncthreads();
    const __nv_bfloat16* Vt = Kst + (t % STAGES) * TK * KROW;
    const int nb = warp * NCOLW;
#pragma unroll
    for (int ks = 0; ks < TK / 16; ++ks) {
      unsigned b[NTW][2];
      if constexpr (NTW == 2) {
        ldsm_x4_t(b[0][0], b[0][1], b[1][0], b[1][1],
                  Vt + (ks * 16 + (lane & 7) + ((lane >> 3) & 1) * 8) * KROW + nb + (lane >> 4) * 8);
      } else {
        ldsm_x2_t(b[0][0], b[0][1], Vt + (ks * 16 + (lane & 7) + ((lane >> 3) & 1) * 8) * KROW + nb);
      }
#pragma unroll
      for (int mt = 0; mt < MT; ++mt) {
        unsigned a0, a1, a2, a3;
        ldsm_x4(a0, a1, a2, a3,
                Pt + (mt * 16 + (lane & 7) + ((lane >> 3) & 1) * 8) * PROW + ks * 16 + (lane >> 4) * 8);
#pragma unroll
        for (int nt = 0; nt < NTW; ++nt) mma_bf16(oacc[mt][nt], a0, a1, a2, a3, b[nt][0], b[nt][1]);
      }
    }
  }
  cp_async_wait<0>();
  __syncthreads();

  // ---- O partial -> smem, cluster reduction through DSMEM ----
  float* Ob = Sb;  // [RP][D]
  {
    const int nb = warp * NCOLW;
#pragma unroll
    for (int mt = 0; mt < MT; ++mt)
#pragma unroll
      for (int nt = 0; nt < NTW; ++nt)
#pragma unroll
        for (int hh = 0; hh < 2; ++hh) {
          const int r = mt * 16 + g4 + hh * 8;
          *reinterpret_cast<float2*>(Ob + r * D + nb + nt * 8 + 2 * t4) =
              make_float2(oacc[mt][nt][hh * 2], oacc[mt][nt][hh * 2 + 1]);
        }
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

template <int D, int MT>
int launch_one(const Params& prm, int C, int num_items, int kv_heads, int smem, cudaStream_t stream) {
  auto kern = attn_mma_kernel<D, MT>;
  static int configured_smem = 0;
  if (smem > configured_smem) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    configured_smem = smem;
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
static bool plan_mma(int D, int MT, int rows, int max_keys, int num_items, int kv_heads, int* C_out,
                     int* chunk_out, int* smem_out);
bool mma_attn_plannable(int dtype, int D, int rows, int max_keys, int num_items, int kv_heads) {
  if (!mma_attn_supported(dtype, D, rows)) return false;
  int C, chunk, smem;
  return plan_mma(D, (rows + 15) / 16, rows, max_keys < 1 ? 1 : max_keys, num_items, kv_heads, &C, &chunk, &smem);
}

// Pick cluster size C and chunk so the whole chunk's logits stay in smem.
static bool plan_mma(int D, int MT, int rows, int max_keys, int num_items, int kv_heads, int* C_out,
                     int* chunk_out, int* smem_out) {
  using namespace mma_attn;
  const int limit = 227 * 1024;
  const int max_tiles = (max_keys + TK - 1) / TK;
  int c_par = (2 * 148 + num_items * kv_heads - 1) / (num_items * kv_heads);  // ~2 CTAs per SM
  c_par = c_par < 1 ? 1 : (c_par > 16 ? 16 : c_par);
  bool found = false;
  for (int C = 1; C <= 16; ++C) {
    int chunk = ((max_tiles + C - 1) / C) * TK;
    if (chunk < TK) chunk = TK;
    const Layout L = make_layout(D, MT, chunk, rows);
    if (L.total > limit) continue;
    *C_out = C;  // smallest fitting C that also gives enough CTAs (or cannot split further)
    *chunk_out = chunk;
    *smem_out = L.total;
    found = true;
    if (C >= c_par || C >= max_tiles) break;
  }
  return found;
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
  int C = 1, chunk = TK, smem = 0;
  if (!plan_mma(D, MT, rows, max_keys < 1 ? 1 : max_keys, num_items, kvp->kv_heads, &C, &chunk, &smem)) return 0;
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
  prm.srow = chunk + 8;
  prm.s_rows = rows;
  *handled = true;
#define SD_MMA_CASE(DD, M) \
  if (D == DD && MT == M) return launch_one<DD, M>(prm, C, num_items, kvp->kv_heads, smem, stream);
  SD_MMA_CASE(128, 1) SD_MMA_CASE(128, 2) SD_MMA_CASE(128, 3) SD_MMA_CASE(128, 4) SD_MMA_CASE(128, 5)
  SD_MMA_CASE(64, 1) SD_MMA_CASE(64, 2) SD_MMA_CASE(64, 3) SD_MMA_CASE(64, 4) SD_MMA_CASE(64, 5)
#undef SD_MMA_CASE
  *handled = false;
  return 0;
}

}  // namespace sd
