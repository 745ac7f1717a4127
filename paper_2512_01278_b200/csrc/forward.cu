// Native layer loop of one batched forward (bf16 weights): the per-layer sequence of
// model.forward_rows (model.py:290-342 restated for R rows at once) issued from C++ so a
// unified iteration costs one host call instead of ~12 Python launches per layer.
//
//   per layer l:  hn = rmsnorm(x)                      sd_rmsnorm_cast (glue.cu)
//                 qkv = hn . Wqkv[l]                   cuBLAS bf16 GEMM, fp32 accumulate
//                 RoPE q/k, K/V -> paged pool          sd_rope_kv_write (K5)
//                 ctx = attention over the work items  sd_attention (K2 verify, K1 draft)
//                 x += ctx . Wo[l]                     cuBLAS, fp32 residual (beta = 1)
//                 hn = rmsnorm(x)
//                 hm = tanh(hn . Win[l])               cuBLAS bf16 + tanh kernel
//                 x += hm . Wout[l]                    cuBLAS, fp32 residual (beta = 1)
//
// Linear layers stay on cuBLAS (north_star: "linear layers may stay on torch matmul").
#include <cublasLt.h>
#include <cublas_v2.h>

#include <map>
#include <mutex>
#include <tuple>
#include <vector>

#include "common.cuh"

extern "C" int sd_rmsnorm_cast(const float* x, int32_t rows, int32_t h, float eps, void* out, int32_t out_dtype,
                               void* stream);
extern "C" int sd_rope_kv_write(const void* qkv, int64_t qkv_row_stride, int32_t rows, const int32_t* row_table,
                                const int32_t* row_pos, const sd_paged_kv* kv, int32_t layer, int32_t q_heads,
                                void* q_out, void* stream);
extern "C" int sd_attention_pair(const void* q, void* out, const sd_paged_kv* kv, int32_t layer,
                                 const sd_attn_launch* verify, const sd_attn_launch* draft, const int32_t* planted,
                                 int32_t num_planted, float planted_bonus, int32_t q_heads, float scale, void* stream);
extern "C" int64_t sd_launch_count(void);
extern "C" int sd_attention(const void* q, void* out, float* lse, const sd_paged_kv* kv, int32_t layer,
                            const int32_t* items, int32_t num_items, int32_t max_keys, int32_t max_nq,
                            const int32_t* crit, uint64_t* acc, int64_t acc_row_stride, int32_t acc_shift,
                            const int32_t* planted, int32_t num_planted, float planted_bonus, int32_t q_heads,
                            float scale, void* workspace, int64_t workspace_bytes, int32_t flags, void* stream);

namespace sd {

__global__ void tanh_bf16_kernel(__nv_bfloat16* x, int64_t n) {
  int64_t i = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * 8;
  const int64_t step = (int64_t)gridDim.x * blockDim.x * 8;
  for (; i + 8 <= n; i += step) {
    uint4 v = *reinterpret_cast<uint4*>(x + i);
    __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&v);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const float2 f = __bfloat1622float2(h[k]);
      h[k] = __floats2bfloat162_rn(tanhf(f.x), tanhf(f.y));
    }
    *reinterpret_cast<uint4*>(x + i) = v;
  }
  if (i < n)
    for (int64_t j = i; j < n; ++j) x[j] = __float2bfloat16_rn(tanhf(__bfloat162float(x[j])));
}

// one handle (+ workspace) per (thread, device): a handle and its workspace are bound to the
// device current at creation
static cublasHandle_t handle_for_thread() {
  constexpr int kMaxDev = 16;
  static thread_local cublasHandle_t hs[kMaxDev] = {};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= kMaxDev) return nullptr;
  cublasHandle_t& h = hs[dev];
  if (h == nullptr) {
    if (cublasCreate(&h) != CUBLAS_STATUS_SUCCESS) return nullptr;
    cublasSetMathMode(h, CUBLAS_DEFAULT_MATH);
    // a 64 MB workspace lets cuBLAS use split-K kernels for the skinny (M ~ 200) GEMMs;
    // owned by the handle for the life of the process (SD_CUBLAS_WS_MB, 0 = none)
    const char* e = getenv("SD_CUBLAS_WS_MB");
    const size_t mb = e && *e ? (size_t)atoi(e) : 64;
    void* ws = nullptr;
    if (mb > 0 && cudaMalloc(&ws, mb << 20) == cudaSuccess) cublasSetWorkspace(h, ws, mb << 20);
  }
  return h;
}

// row-major C[R x N] (+)= A[R x K] . W with W stored [N][K] (out-major, nn.Linear layout):
// column-major C^T = op_T(W) . A^T, i.e. cuBLAS's TN form.  A, W bf16; C bf16 or fp32
// (beta = 0 / 1).
//
// cuBLASLt with an algorithm chosen per (rows rounded up to 16, N, K, C type, beta) by
// timing the heuristic's candidates once (synchronously, on first use; the bench's
// untimed pre-roll meets every bucket it later times): for the skinny decode shapes the
// default heuristic leaves up to 20% on the table (mlp_in at 228 rows: 31.6 -> 25.4 us,
// tools/lt_probe.cu).  SD_GEMM_TUNE=0 keeps plain cublasGemmEx.
struct LtPlan {
  cublasLtMatmulAlgo_t algo;
  bool valid = false;
};
struct LtState {
  cublasLtHandle_t lt = nullptr;
  void* ws = nullptr;
  size_t ws_bytes = 0;
  std::map<std::tuple<int, int, int, int, int>, LtPlan> plans;
};
static LtState* lt_state() {
  constexpr int kMaxDev = 16;
  static thread_local LtState st[kMaxDev];
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= kMaxDev) return nullptr;
  LtState& a = st[dev];
  if (a.lt == nullptr) {
    if (cublasLtCreate(&a.lt) != CUBLAS_STATUS_SUCCESS) return nullptr;
    a.ws_bytes = 64u << 20;
    if (cudaMalloc(&a.ws, a.ws_bytes) != cudaSuccess) a.ws = nullptr, a.ws_bytes = 0;
  }
  return &a;
}

struct LtCall {
  cublasLtMatmulDesc_t op = nullptr;
  cublasLtMatrixLayout_t la = nullptr, lb = nullptr, lc = nullptr;
  ~LtCall() {
    if (op) cublasLtMatmulDescDestroy(op);
    if (la) cublasLtMatrixLayoutDestroy(la);
    if (lb) cublasLtMatrixLayoutDestroy(lb);
    if (lc) cublasLtMatrixLayoutDestroy(lc);
  }
  bool init(int R, int N, int K, bool c_f32) {
    if (cublasLtMatmulDescCreate(&op, CUBLAS_COMPUTE_32F, CUDA_R_32F) != CUBLAS_STATUS_SUCCESS) return false;
    const cublasOperation_t ta = CUBLAS_OP_T, tb = CUBLAS_OP_N;
    cublasLtMatmulDescSetAttribute(op, CUBLASLT_MATMUL_DESC_TRANSA, &ta, sizeof(ta));
    cublasLtMatmulDescSetAttribute(op, CUBLASLT_MATMUL_DESC_TRANSB, &tb, sizeof(tb));
    return cublasLtMatrixLayoutCreate(&la, CUDA_R_16BF, K, N, K) == CUBLAS_STATUS_SUCCESS &&
           cublasLtMatrixLayoutCreate(&lb, CUDA_R_16BF, K, R, K) == CUBLAS_STATUS_SUCCESS &&
           cublasLtMatrixLayoutCreate(&lc, c_f32 ? CUDA_R_32F : CUDA_R_16BF, N, R, N) == CUBLAS_STATUS_SUCCESS;
  }
};

// time the heuristic candidates for rows Rb on scratch buffers; returns the fastest
static LtPlan lt_tune(LtState* st, int Rb, int N, int K, bool c_f32, float beta, cudaStream_t s) {
  LtPlan plan;
  LtCall call;
  if (!call.init(Rb, N, K, c_f32)) return plan;
  cublasLtMatmulPreference_t pref;
  if (cublasLtMatmulPreferenceCreate(&pref) != CUBLAS_STATUS_SUCCESS) return plan;
  cublasLtMatmulPreferenceSetAttribute(pref, CUBLASLT_MATMUL_PREF_MAX_WORKSPACE_BYTES, &st->ws_bytes,
                                       sizeof(st->ws_bytes));
  static const int max_cand = [] {
    const char* v = getenv("SD_GEMM_CANDIDATES");
    return std::max(1, std::min(64, v && *v ? atoi(v) : 8));
  }();
  cublasLtMatmulHeuristicResult_t res[64];
  int n = 0;
  cublasLtMatmulAlgoGetHeuristic(st->lt, call.op, call.la, call.lb, call.lc, call.lc, pref, max_cand, res, &n);
  cublasLtMatmulPreferenceDestroy(pref);
  void *A = nullptr, *W = nullptr, *C = nullptr;
  const size_t cb = (size_t)Rb * N * (c_f32 ? 4 : 2);
  if (n <= 0 || cudaMalloc(&A, (size_t)Rb * K * 2) != cudaSuccess || cudaMalloc(&W, (size_t)N * K * 2) != cudaSuccess ||
      cudaMalloc(&C, cb) != cudaSuccess) {
    cudaFree(A), cudaFree(W), cudaFree(C);
    cudaGetLastError();
    return plan;
  }
  cudaMemsetAsync(A, 0, (size_t)Rb * K * 2, s);
  cudaMemsetAsync(W, 0, (size_t)N * K * 2, s);
  cudaMemsetAsync(C, 0, cb, s);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0), cudaEventCreate(&e1);
  const float alpha = 1.f;
  float best = 1e30f;
  for (int i = 0; i < n; ++i) {
    if (res[i].state != CUBLAS_STATUS_SUCCESS) continue;
    bool ok = true;
    float tot = 0.f;
    for (int it = 0; it < 6 && ok; ++it) {
      cudaEventRecord(e0, s);
      ok = cublasLtMatmul(st->lt, call.op, &alpha, W, call.la, A, call.lb, &beta, C, call.lc, C, call.lc, &res[i].algo,
                          st->ws, st->ws_bytes, s) == CUBLAS_STATUS_SUCCESS;
      cudaEventRecord(e1, s);
      cudaEventSynchronize(e1);
      float ms = 0.f;
      cudaEventElapsedTime(&ms, e0, e1);
      if (it >= 2) tot += ms;  // first runs warm the kernel up
    }
    if (ok && tot < best) best = tot, plan.algo = res[i].algo, plan.valid = true;
  }
  cudaEventDestroy(e0), cudaEventDestroy(e1);
  cudaStreamSynchronize(s);
  cudaFree(A), cudaFree(W), cudaFree(C);
  cudaGetLastError();
  return plan;
}

static int gemm_tune_enabled() {
  static const int tune = [] {
    const char* v = getenv("SD_GEMM_TUNE");
    return v && *v ? atoi(v) : 1;
  }();
  return tune;
}

// the tuned plan of one GEMM shape, created on first use (tuning synchronises: never
// inside a stream capture, see gemm_prepare)
static const LtPlan* gemm_plan(cublasHandle_t hd, int R, int N, int K, bool c_f32, float beta) {
  LtState* st = lt_state();
  if (st == nullptr || st->ws == nullptr) return nullptr;
  cudaStream_t s = nullptr;
  cublasGetStream(hd, &s);
  const int Rb = (R + 15) / 16 * 16;
  const auto key = std::make_tuple(Rb, N, K, c_f32 ? 1 : 0, beta != 0.f ? 1 : 0);
  auto it = st->plans.find(key);
  if (it == st->plans.end()) it = st->plans.emplace(key, lt_tune(st, Rb, N, K, c_f32, beta, s)).first;
  return &it->second;
}

static void gemm_prepare(cublasHandle_t hd, int R, int N, int K, bool c_f32, float beta) {
  if (gemm_tune_enabled()) gemm_plan(hd, R, N, K, c_f32, beta);
}

static int gemm(cublasHandle_t hd, int R, int N, int K, const void* A, const void* Wt, void* C, bool c_f32,
                float beta) {
  const float alpha = 1.f;
  if (gemm_tune_enabled()) {
    const LtPlan* plan = gemm_plan(hd, R, N, K, c_f32, beta);
    if (plan != nullptr && plan->valid) {
      LtState* st = lt_state();
      cudaStream_t s = nullptr;
      cublasGetStream(hd, &s);
      LtCall call;
      cublasLtMatmulHeuristicResult_t chk;
      if (call.init(R, N, K, c_f32) &&
          cublasLtMatmulAlgoCheck(st->lt, call.op, call.la, call.lb, call.lc, call.lc, &plan->algo, &chk) ==
              CUBLAS_STATUS_SUCCESS &&
          cublasLtMatmul(st->lt, call.op, &alpha, Wt, call.la, A, call.lb, &beta, C, call.lc, C, call.lc, &plan->algo,
                         st->ws, st->ws_bytes, s) == CUBLAS_STATUS_SUCCESS)
        return 0;
    }
  }
  const cublasStatus_t st =
      cublasGemmEx(hd, CUBLAS_OP_T, CUBLAS_OP_N, N, R, K, &alpha, Wt, CUDA_R_16BF, K, A, CUDA_R_16BF, K, &beta, C,
                   c_f32 ? CUDA_R_32F : CUDA_R_16BF, N, CUBLAS_COMPUTE_32F, CUBLAS_GEMM_DEFAULT);
  if (st != CUBLAS_STATUS_SUCCESS) {
    set_error("sd_forward_layers: cublasGemmEx failed (" + std::to_string((int)st) + ")");
    return -1;
  }
  return 0;
}

// Side streams for the attention launches of one layer: the verify launch (K2) on a
// high-priority stream, the draft launch (K1) on a low-priority one, both forked from and
// joined back into the caller's stream, so the block scheduler hands free CTA slots to K2
// first and K1's CTAs fill K2's tail waves (one per (thread, device)).
struct AttnStreams {
  cudaStream_t hi = nullptr, lo = nullptr;
  cudaEvent_t fork = nullptr, join_hi = nullptr, join_lo = nullptr;
};

static AttnStreams* attn_streams() {
  constexpr int kMaxDev = 16;
  static thread_local AttnStreams st[kMaxDev];
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= kMaxDev) return nullptr;
  AttnStreams& a = st[dev];
  if (a.hi == nullptr) {
    int least = 0, greatest = 0;
    cudaDeviceGetStreamPriorityRange(&least, &greatest);
    if (cudaStreamCreateWithPriority(&a.hi, cudaStreamNonBlocking, greatest) != cudaSuccess ||
        cudaStreamCreateWithPriority(&a.lo, cudaStreamNonBlocking, least) != cudaSuccess ||
        cudaEventCreateWithFlags(&a.fork, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&a.join_hi, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&a.join_lo, cudaEventDisableTiming) != cudaSuccess) {
      cudaGetLastError();
      a = AttnStreams{};
      return nullptr;
    }
  }
  return &a;
}

}  // namespace sd

namespace {
int attn_launch(const sd_attn_launch& a, const void* q, void* ctx, const sd_paged_kv* kv, int l,
                const int32_t* planted, int32_t num_planted, float planted_bonus, int32_t q_heads, float scale,
                void* workspace, int64_t workspace_bytes, cudaStream_t s) {
  return sd_attention(q, ctx, nullptr, kv, l, a.items, a.num_items, a.max_keys, a.max_nq, a.crit, a.acc,
                      a.acc_row_stride, a.acc_shift, planted, num_planted, planted_bonus, q_heads, scale, workspace,
                      workspace_bytes, 0, s);
}
}  // namespace

extern "C" int64_t sd_forward_workspace_bytes(int32_t rows, int32_t head_dim, int64_t attention_bytes) {
  return ((attention_bytes + 255) / 256) * 256 + sd::rope_table_bytes(rows, head_dim) + 256;  // + alignment slack
}

namespace {
// everything one forward issues on stream s (and the two attention side streams)
struct LayerLoop {
  const sd_layer_weights* w;
  int32_t layers;
  float* x;
  void *hn, *qkv, *q, *ctx, *hm;
  int32_t rows, hidden, q_heads;
  const int32_t *row_table, *row_pos;
  const sd_paged_kv* kv;
  const sd_attn_launch* launches;
  int32_t num_launches;
  const int32_t* planted;
  int32_t num_planted;
  float planted_bonus, scale, eps;
  void* workspace;
  int64_t workspace_bytes;
  void* const* attn_events;
  int32_t flags;
  void* stream;
  int l0 = 0, l1 = -1;  // layer range to issue ([0, layers) when l1 < 0)
};

int issue_layers(const LayerLoop& a, cublasHandle_t hd) {
  cudaStream_t s = static_cast<cudaStream_t>(a.stream);
  void* stream = a.stream;
  const sd_paged_kv* kv = a.kv;
  const sd_attn_launch* launches = a.launches;
  const int num_launches = a.num_launches, rows = a.rows, hidden = a.hidden, q_heads = a.q_heads;
  float* x = a.x;
  void* workspace = a.workspace;
  int64_t workspace_bytes = a.workspace_bytes;
  const int qkv_w = (q_heads + 2 * kv->kv_heads) * kv->head_dim;
  const int64_t hm_n = (int64_t)rows * 2 * hidden;
  const int tanh_blocks = (int)std::min<int64_t>((hm_n / 8 + 255) / 256 + 1, 148 * 8);
  // RoPE cos/sin of every row once for all layers, at the end of the workspace
  // (sd_forward_workspace_bytes); the attention launches get the rest
  const int64_t table_bytes = sd::rope_table_bytes(rows, kv->head_dim);
  // the table's start is 256-byte aligned (the K5 kernel reads it in 16-byte vectors)
  const uintptr_t ws0 = reinterpret_cast<uintptr_t>(workspace);
  const uintptr_t tab0 = workspace != nullptr ? ((ws0 + workspace_bytes - table_bytes) & ~uintptr_t(255)) : 0;
  const bool use_table = kv->head_dim % 16 == 0 && (qkv_w % 8) == 0 && workspace != nullptr &&
                         workspace_bytes >= table_bytes + 256 && tab0 >= ws0;
  float2* table = nullptr;
  const int l0 = a.l0, l1 = a.l1 < 0 ? a.layers : a.l1;
  if (use_table) {
    workspace_bytes = (int64_t)(tab0 - ws0);
    table = reinterpret_cast<float2*>(tab0);
    if (l0 == 0) sd::rope_table(a.row_pos, rows, kv->head_dim, table, s);  // kept for later layer ranges
  }
  // two attention launches (verify + draft) overlap on priority streams unless timed per
  // launch (attn_events) or disabled (flags bit 0)
  sd::AttnStreams* as = nullptr;
  const bool overlap = num_launches == 2 && a.attn_events == nullptr && !(a.flags & 1) &&
                       launches[0].num_items > 0 && launches[1].num_items > 0 && (as = sd::attn_streams()) != nullptr;
  // f3 fused verify + draft launch (flags bit 1): launch 0 dense verify, launch 1 drafts
  const bool fused = (a.flags & 2) && num_launches == 2 && a.attn_events == nullptr && launches[0].num_items > 0 &&
                     launches[1].num_items > 0 && launches[0].crit == nullptr && launches[1].crit != nullptr &&
                     launches[1].max_nq == 1;
  const void* q = a.q;
  void* ctx = a.ctx;
  int rc;
  for (int l = l0; l < l1; ++l) {
    const sd_layer_weights& wl = a.w[l];
    if ((rc = sd_rmsnorm_cast(x, rows, hidden, a.eps, a.hn, SD_DTYPE_BF16, stream)) != 0) return rc;
    if ((rc = sd::gemm(hd, rows, qkv_w, hidden, a.hn, wl.w_qkv, a.qkv, false, 0.f)) != 0) return rc;
    if (use_table)
      sd::rope_kv_write_table(a.qkv, qkv_w, rows, a.row_table, a.row_pos, kv, l, q_heads, table, a.q, s);
    else if ((rc = sd_rope_kv_write(a.qkv, qkv_w, rows, a.row_table, a.row_pos, kv, l, q_heads, a.q, stream)) != 0)
      return rc;
    if (fused) {
      // f3: one launch, the verify grid's CTAs take the draft units after their verify chunk
      rc = sd_attention_pair(q, ctx, kv, l, &launches[0], &launches[1], a.planted, a.num_planted, a.planted_bonus,
                             q_heads, a.scale, stream);
      if (rc == 0) goto attn_done;
      if (rc != 1) return rc;
    }
    if (overlap) {
      // K2 (launch 0) high priority, K1 (launch 1) low priority, concurrently
      cudaEventRecord(as->fork, s);
      cudaStreamWaitEvent(as->hi, as->fork, 0);
      cudaStreamWaitEvent(as->lo, as->fork, 0);
      if ((rc = attn_launch(launches[0], q, ctx, kv, l, a.planted, a.num_planted, a.planted_bonus, q_heads, a.scale,
                            workspace, workspace_bytes, as->hi)) != 0)
        return rc;
      if ((rc = attn_launch(launches[1], q, ctx, kv, l, a.planted, a.num_planted, a.planted_bonus, q_heads, a.scale,
                            workspace, workspace_bytes, as->lo)) != 0)
        return rc;
      cudaEventRecord(as->join_hi, as->hi);
      cudaEventRecord(as->join_lo, as->lo);
      cudaStreamWaitEvent(s, as->join_hi, 0);
      cudaStreamWaitEvent(s, as->join_lo, 0);
    } else {
      for (int i = 0; i < num_launches; ++i) {
        const sd_attn_launch& al = launches[i];
        if (al.num_items == 0) continue;
        cudaEvent_t* ev =
            a.attn_events ? (cudaEvent_t*)(a.attn_events + 2 * ((int64_t)l * num_launches + i)) : nullptr;
        if (ev && ev[0]) cudaEventRecord(ev[0], s);
        if ((rc = attn_launch(al, q, ctx, kv, l, a.planted, a.num_planted, a.planted_bonus, q_heads, a.scale,
                              workspace, workspace_bytes, s)) != 0)
          return rc;
        if (ev && ev[1]) cudaEventRecord(ev[1], s);
      }
    }
  attn_done:
    if ((rc = sd::gemm(hd, rows, hidden, hidden, ctx, wl.wo, x, true, 1.f)) != 0) return rc;
    if ((rc = sd_rmsnorm_cast(x, rows, hidden, a.eps, a.hn, SD_DTYPE_BF16, stream)) != 0) return rc;
    if ((rc = sd::gemm(hd, rows, 2 * hidden, hidden, a.hn, wl.mlp_in, a.hm, false, 0.f)) != 0) return rc;
    sd::tanh_bf16_kernel<<<tanh_blocks, 256, 0, s>>>(static_cast<__nv_bfloat16*>(a.hm), hm_n);
    sd::count_launch();
    if ((rc = sd::gemm(hd, rows, hidden, 2 * hidden, a.hm, wl.mlp_out, x, true, 1.f)) != 0) return rc;
  }
  // the workspace is handed back zero-filled (the attention launches rely on it)
  if (use_table && l1 == a.layers) cudaMemsetAsync(table, 0, table_bytes, s);
  return 0;
}

// The forward as one CUDA graph (flags bit 3): the layer loop is captured on the caller's
// stream (side streams join the capture through the fork / join events), the capture is
// applied to a cached executable graph with cudaGraphExecUpdate (same topology: only
// kernel parameters and grids changed since the last iteration; re-instantiated when
// the topology changed), and launched.  Two executables alternate so an update never
// touches the one the previous, possibly still running, iteration launched.  The host
// cost is the capture (~ the eager enqueue) + the update; the device runs the ~300
// launches without per-launch front-end gaps.
constexpr int kGraphChunks = 3;
struct GraphCache {
  cudaGraphExec_t exec[kGraphChunks][2] = {};
  std::vector<unsigned> sig[kGraphChunks][2];  // cluster shape of every kernel node of the executable
  int next[kGraphChunks] = {};
  int64_t instantiations = 0, updates = 0;
  // captured and launched on an own stream (the caller's may be the legacy default stream,
  // which cannot be captured), ordered after / before the caller's work by events
  cudaStream_t cs = nullptr;
  cudaEvent_t in = nullptr, out = nullptr;
};
GraphCache* graph_cache() {
  constexpr int kMaxDev = 16;
  static thread_local GraphCache gc[kMaxDev];
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= kMaxDev) return nullptr;
  return &gc[dev];
}

// Capture one layer range on the graph stream s, apply it to chunk `ci`'s cached executable
// and launch it.  0: launched; 1: not capturable (nothing of it ran); < 0: error.
int capture_chunk(GraphCache* gc, int ci, const LayerLoop& ac, cublasHandle_t hd) {
  cudaStream_t s = static_cast<cudaStream_t>(ac.stream);
  if (cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal) != cudaSuccess) {
    cudaGetLastError();
    return 1;
  }
  const int64_t launches0 = sd_launch_count();
  const int rc = issue_layers(ac, hd);
  cudaGraph_t g = nullptr;
  const cudaError_t ce = cudaStreamEndCapture(s, &g);
  if (rc != 0 || ce != cudaSuccess || g == nullptr) {
    if (g) cudaGraphDestroy(g);
    cudaGetLastError();
    sd::count_launch(-(int)(sd_launch_count() - launches0));  // nothing of the capture ran
    return rc < 0 ? rc : 1;
  }
  // an in-place update keeps the executable's launch attributes: the cluster shape of every
  // kernel node (the K2 planner's cluster size varies with the context) must match
  std::vector<unsigned> sig;
  {
    size_t n = 0;
    cudaGraphGetNodes(g, nullptr, &n);
    std::vector<cudaGraphNode_t> nodes(n);
    cudaGraphGetNodes(g, nodes.data(), &n);
    sig.reserve(n);
    for (size_t i = 0; i < n; ++i) {
      cudaGraphNodeType t;
      cudaGraphNodeGetType(nodes[i], &t);
      unsigned v = 0xffffffffu;
      if (t == cudaGraphNodeTypeKernel) {
        cudaLaunchAttributeValue av{};
        v = cudaGraphKernelNodeGetAttribute(nodes[i], cudaLaunchAttributeClusterDimension, &av) == cudaSuccess
                ? av.clusterDim.x * 65536u + av.clusterDim.y * 256u + av.clusterDim.z
                : 0u;
      }
      sig.push_back(v);
    }
    cudaGetLastError();
  }
  static const int allow_update = [] {
    const char* v = getenv("SD_GRAPH_UPDATE");
    return v && *v ? atoi(v) : 1;
  }();
  const int slot = gc->next[ci];
  cudaGraphExec_t& ex = gc->exec[ci][slot];
  gc->next[ci] ^= 1;
  if (ex != nullptr && (!allow_update || gc->sig[ci][slot] != sig)) {
    cudaGraphExecDestroy(ex);
    ex = nullptr;
  }
  if (ex != nullptr) {
    cudaGraphExecUpdateResultInfo info;
    if (cudaGraphExecUpdate(ex, g, &info) == cudaSuccess) {
      ++gc->updates;
    } else {
      cudaGetLastError();
      cudaGraphExecDestroy(ex);
      ex = nullptr;
    }
  }
  if (ex == nullptr) {
    if (cudaGraphInstantiate(&ex, g, 0) != cudaSuccess) {
      cudaGetLastError();
      ex = nullptr;
      cudaGraphDestroy(g);
      sd::count_launch(-(int)(sd_launch_count() - launches0));
      return 1;
    }
    ++gc->instantiations;
    gc->sig[ci][slot] = std::move(sig);
  }
  cudaGraphDestroy(g);
  if (cudaGraphLaunch(ex, s) != cudaSuccess) {
    sd::set_error("sd_forward_layers: cudaGraphLaunch failed");
    return -1;
  }
  return 0;
}

// The layer stack as CUDA graphs of three layer ranges, [0, 2), [2, 8), [8, L): the first
// range's capture is short, so after an idle stream (the first iteration of a pipeline)
// the GPU starts within ~0.1 ms while the host captures the rest, instead of waiting for
// the whole ~2 ms capture.  0: launched; 1: nothing launched (caller issues directly); < 0 error
int launch_as_graph(const LayerLoop& a, cublasHandle_t hd) {
  GraphCache* gc = graph_cache();
  if (gc == nullptr) return 1;
  if (gc->cs == nullptr) {
    if (cudaStreamCreateWithFlags(&gc->cs, cudaStreamNonBlocking) != cudaSuccess ||
        cudaEventCreateWithFlags(&gc->in, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&gc->out, cudaEventDisableTiming) != cudaSuccess) {
      cudaGetLastError();
      gc->cs = nullptr;
      return 1;
    }
  }
  cudaStream_t caller = static_cast<cudaStream_t>(a.stream);
  cudaStream_t s = gc->cs;
  // every cuBLASLt plan this forward needs is tuned before the capture (tuning synchronises)
  const int qkv_w = (a.q_heads + 2 * a.kv->kv_heads) * a.kv->head_dim;
  sd::gemm_prepare(hd, a.rows, qkv_w, a.hidden, false, 0.f);
  sd::gemm_prepare(hd, a.rows, a.hidden, a.hidden, true, 1.f);
  sd::gemm_prepare(hd, a.rows, 2 * a.hidden, a.hidden, false, 0.f);
  sd::gemm_prepare(hd, a.rows, a.hidden, 2 * a.hidden, true, 1.f);
  if (sd::attn_streams() == nullptr) return 1;
  cudaGetLastError();
  static const int chunked = [] {
    const char* v = getenv("SD_GRAPH_CHUNKS");
    return v && *v ? atoi(v) : 1;
  }();
  const int bounds[kGraphChunks + 1] = {0, chunked ? std::min(2, a.layers) : 0, chunked ? std::min(8, a.layers) : 0,
                                        a.layers};
  // the graph stream waits for the caller's prior work (outside the captures)
  cudaEventRecord(gc->in, caller);
  cudaStreamWaitEvent(s, gc->in, 0);
  cublasSetStream(hd, s);
  int rc = 0;
  int ci = 0;
  for (; ci < kGraphChunks && rc == 0; ++ci) {
    if (bounds[ci] == bounds[ci + 1]) continue;
    LayerLoop ac = a;
    ac.stream = s;
    ac.l0 = bounds[ci], ac.l1 = bounds[ci + 1];
    rc = capture_chunk(gc, ci, ac, hd);
    if (rc == 1) {
      // not capturable: the rest of the stack goes out directly, still on the graph stream
      LayerLoop ar = a;
      ar.stream = s;
      ar.l0 = bounds[ci];
      rc = issue_layers(ar, hd);
      break;
    }
  }
  cublasSetStream(hd, caller);
  if (rc != 0) return rc < 0 ? rc : -1;
  // the caller's later work waits for the graphs
  cudaEventRecord(gc->out, s);
  cudaStreamWaitEvent(caller, gc->out, 0);
  return 0;
}
}  // namespace

extern "C" int sd_forward_layers(const sd_layer_weights* w, int32_t layers, float* x, void* hn, void* qkv, void* q,
                                 void* ctx, void* hm, int32_t rows, int32_t hidden, int32_t q_heads,
                                 const int32_t* row_table, const int32_t* row_pos, const sd_paged_kv* kv,
                                 const sd_attn_launch* launches, int32_t num_launches, const int32_t* planted,
                                 int32_t num_planted, float planted_bonus, float scale, float eps, void* workspace,
                                 int64_t workspace_bytes, void* const* attn_events, int32_t flags, void* stream) {
  SD_REQUIRE(w != nullptr && x != nullptr && kv != nullptr, "sd_forward_layers: null pointer");
  SD_REQUIRE(kv->dtype == SD_DTYPE_BF16, "sd_forward_layers: bf16 pools only (fp32 parity mode runs in torch)");
  SD_REQUIRE(rows > 0 && layers > 0 && num_launches >= 0, "sd_forward_layers: bad sizes");
  cublasHandle_t hd = sd::handle_for_thread();
  SD_REQUIRE(hd != nullptr, "sd_forward_layers: cublasCreate failed");
  cublasSetStream(hd, static_cast<cudaStream_t>(stream));
  const LayerLoop a{w,        layers,          x,         hn,      qkv,         q,          ctx,
                    hm,       rows,            hidden,    q_heads, row_table,   row_pos,    kv,
                    launches, num_launches,    planted,   num_planted, planted_bonus, scale, eps,
                    workspace, workspace_bytes, attn_events, flags, stream};
  int rc = 1;
  // flags bit 3: one CUDA graph for the whole loop (not with per-launch timing events).
  // (Direct launches whenever the stream is idle, since they start running as they are
  // issued, measured slower: 3129 vs 3157 tok/s over 5-iteration windows.)
  const bool use_graph = (flags & 8) && attn_events == nullptr;
  if (use_graph) rc = launch_as_graph(a, hd);
  if (rc == 1) rc = issue_layers(a, hd);
  if (rc != 0) return rc;
  SD_CUDA_RETURN();
}

extern "C" int64_t sd_forward_graph_stats(int32_t which) {
  GraphCache* gc = graph_cache();
  if (gc == nullptr) return -1;
  return which == 0 ? gc->instantiations : gc->updates;
}

// One linear layer through the same tuned path (the LM head of the batched forward):
// C[R][N] (+)= A[R][K] . W^T, A / W bf16, C fp32 (c_f32) or bf16, beta 0 or 1.
extern "C" int sd_linear(const void* A, const void* W, void* C, int32_t R, int32_t N, int32_t K, int32_t c_f32,
                         float beta, void* stream) {
  SD_REQUIRE(A != nullptr && W != nullptr && C != nullptr, "sd_linear: null pointer");
  SD_REQUIRE(R > 0 && N > 0 && K > 0, "sd_linear: bad sizes");
  cublasHandle_t hd = sd::handle_for_thread();
  SD_REQUIRE(hd != nullptr, "sd_linear: cublasCreate failed");
  cublasSetStream(hd, static_cast<cudaStream_t>(stream));
  const int rc = sd::gemm(hd, R, N, K, A, W, C, c_f32 != 0, beta);
  if (rc != 0) return rc;
  SD_CUDA_RETURN();
}
