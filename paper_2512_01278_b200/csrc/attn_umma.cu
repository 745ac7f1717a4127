// tcgen05 attention dispatch for sm_100a: the head-packed K1 draft kernel (this file), the
// K2 verify kernel (attn_umma.cuh, instantiated per GQA group in attn_umma_g4/g8.cu) and
// the launch planner that picks the cluster split.
#include "attn_umma.cuh"

#include <atomic>
#include <map>
#include <mutex>
#include <algorithm>
#include <tuple>

#include <cuda.h>

namespace sd {
namespace umma_attn {

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
  // K1 head packing: four kv heads per CTA (32-key tiles) while the critical list fits the
  // TMEM-resident logits, else two heads per CTA (64-key tiles: twice the keys resident),
  // else the clustered verify kernel over the gathered keys (SD_UMMA_HPC forces one packing)
  static const int hpc_env = env_int("SD_UMMA_HPC", 0);
  for (int HPC : {4, 2}) {
    if (!hp_env || max_nq != 1 || kvp->dtype != SD_DTYPE_BF16 || kvp->head_dim != D || !(G == 4 || G == 8) ||
        kvp->kv_heads % HPC != 0 || (hpc_env && hpc_env != HPC))
      continue;
    const int KPT = TK / HPC;
    const int NQ = HPC * G, NR = NQ < 16 ? 16 : NQ, tmax = (256 - NR) / NR;
    const int ct_tiles = (max(max_keys, 1) + KPT - 1) / KPT;  // KPT-key tiles
    const int ct = (ct_tiles * KPT + TK - 1) / TK;           // 128-key units for the staging arrays
    if (ct_tiles > tmax || make_hp_layout(NR, 2, tmax, ct).total > 113 * 1024) continue;  // logits stay resident
    prm.chunk = ct * TK;
    *handled = true;
    // a third 32 KB ring slot when two CTAs per SM still fit (deeper loads in flight)
    static const int hp_slots = env_int("SD_UMMA_HP_SLOTS", 3);
    const bool three = hp_slots == 3 && make_hp_layout(NR, 3, tmax, ct).total <= 113 * 1024;
    if (HPC == 2) {
      if (G == 4)
        return three ? launch_hp<4, 2, 3, 256>(prm, num_items, kvp->kv_heads, ct, stream)
                     : launch_hp<4, 2, 2, 256>(prm, num_items, kvp->kv_heads, ct, stream);
      return three ? launch_hp<8, 2, 3, 256>(prm, num_items, kvp->kv_heads, ct, stream)
                   : launch_hp<8, 2, 2, 256>(prm, num_items, kvp->kv_heads, ct, stream);
    }
    if (G == 4)
      return three ? launch_hp<4, 4, 3, 256>(prm, num_items, kvp->kv_heads, ct, stream)
                   : launch_hp<4, 4, 2, 256>(prm, num_items, kvp->kv_heads, ct, stream);
    return three ? launch_hp<8, 4, 3, 256>(prm, num_items, kvp->kv_heads, ct, stream)
                 : launch_hp<8, 4, 2, 256>(prm, num_items, kvp->kv_heads, ct, stream);
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

// f3: one fused launch for a layer's verify items (dense, score emission) and draft items
// (critical list, one query token): the verify clusters' CTAs claim the draft units once
// their verify chunk is done (attn_fused_kernel).  Returns 1 without launching when the
// shapes do not qualify (the caller launches the two separately), 0 on success.
int launch_attn_pair(const void* q, void* out, const sd_paged_kv* kvp, int layer, const int32_t* v_items, int v_n,
                     int v_keys, int v_nq, unsigned long long* v_acc, int64_t v_acc_stride, int v_acc_shift,
                     const int32_t* d_items, int d_n, int d_keys, const int32_t* d_crit, const int32_t* planted,
                     int n_planted, float bonus, int q_heads, float scale, cudaStream_t stream) {
  using namespace umma_attn;
  const int G = q_heads / kvp->kv_heads;
  if (v_n < 1 || d_n < 1 || d_crit == nullptr || kvp->dtype != SD_DTYPE_BF16 || kvp->head_dim != D ||
      !(G == 4 || G == 8) || kvp->kv_heads % 4 != 0 || kvp->page_shift < 4 || env_int("SD_ATTN_TRACE", 0))
    return 1;
  UmmaPlan pl;
  if (!umma_plan(kvp, v_n, v_keys, v_nq, q_heads, 1, &pl) || pl.NR > kNarrowMaxNR) return 1;
  const int NRd = 4 * G, tmax = (256 - NRd) / NRd;
  const int ct_tiles = (max(d_keys, 1) + 31) / 32;
  const int ct = (ct_tiles * 32 + TK - 1) / TK;
  if (ct_tiles > tmax) return 1;
  const int Sv = 256 / pl.NR;
  const int smem = std::max(make_layout(pl.NR, 2, Sv, pl.chunk / TK, 1).total, make_hp_layout(NRd, 2, tmax, ct).total);
  if (smem > 113 * 1024) return 1;
  static std::mutex mu;
  static unsigned int* ctr[64] = {};
  static int parity[64] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  int par;
  {
    std::lock_guard<std::mutex> lock(mu);
    if (ctr[dev & 63] == nullptr) {
      if (cudaMalloc(&ctr[dev & 63], 4 * sizeof(unsigned int)) != cudaSuccess) return 1;
      cudaMemset(ctr[dev & 63], 0, 4 * sizeof(unsigned int));
    }
    par = parity[dev & 63];
    parity[dev & 63] ^= 1;
  }
  Params pv{}, pd{};
  pv.q = pd.q = static_cast<const __nv_bfloat16*>(q);
  pv.out = pd.out = static_cast<__nv_bfloat16*>(out);
  pv.kv = pd.kv = make_paged(kvp);
  pv.layer = pd.layer = layer;
  pv.planted = pd.planted = planted;
  pv.n_planted = pd.n_planted = n_planted;
  pv.bonus_log2 = pd.bonus_log2 = bonus * LOG2E;
  pv.q_heads = pd.q_heads = q_heads;
  pv.scale_log2 = pd.scale_log2 = scale * LOG2E;
  pv.items = v_items;
  pv.acc = v_acc;
  pv.acc_stride = v_acc_stride;
  pv.acc_scale = ldexpf(1.f, v_acc_shift);
  pv.chunk = pl.chunk;
  pv.dense = 1;
  static const int tma_env = env_int("SD_K2_TMA", 1);
  if (tma_env) {
    const int64_t loff = (int64_t)layer * kvp->layer_stride * 2;
    pv.tma = pool_map(&pv.tmk, static_cast<const char*>(kvp->k) + loff, kvp->num_slots, kvp->kv_heads) &&
             pool_map(&pv.tmv, static_cast<const char*>(kvp->v) + loff, kvp->num_slots, kvp->kv_heads);
  }
  pd.items = d_items;
  pd.crit = d_crit;
  pd.chunk = ct * TK;
  static const int any_cta = env_int("SD_FUSED_ANY", 0);
  FusedCtl fc{ctr[dev & 63], par, d_n * (kvp->kv_heads / 4), kvp->kv_heads / 4, pl.C * kvp->kv_heads * v_n, any_cta};
  const int rc = G == 4 ? launch_fused_g4(pv, pd, fc, pl.NR, pl.C, v_n, kvp->kv_heads, smem, stream)
                        : launch_fused_g8(pv, pd, fc, pl.NR, pl.C, v_n, kvp->kv_heads, smem, stream);
  return rc < 0 ? 1 : rc;
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

// f3 fused verify + draft launch through the C ABI (csrc/attn_umma.cu launch_attn_pair):
// returns 1 when the pair does not qualify (launch the two with sd_attention instead).
extern "C" int sd_attention_pair(const void* q, void* out, const sd_paged_kv* kv, int32_t layer,
                                 const sd_attn_launch* verify, const sd_attn_launch* draft, const int32_t* planted,
                                 int32_t num_planted, float planted_bonus, int32_t q_heads, float scale, void* stream) {
  SD_REQUIRE(q != nullptr && out != nullptr && kv != nullptr && verify != nullptr && draft != nullptr,
             "sd_attention_pair: null pointer");
  SD_REQUIRE(kv->kv_heads > 0 && q_heads % kv->kv_heads == 0, "sd_attention_pair: kv_heads must divide q_heads");
  return sd::launch_attn_pair(q, out, kv, layer, verify->items, verify->num_items, verify->max_keys, verify->max_nq,
                              reinterpret_cast<unsigned long long*>(verify->acc), verify->acc_row_stride,
                              verify->acc_shift, draft->items, draft->num_items, draft->max_keys, draft->crit, planted,
                              num_planted, planted_bonus, q_heads, scale, static_cast<cudaStream_t>(stream));
}
