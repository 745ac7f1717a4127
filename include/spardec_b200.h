/*
 * spardec_b200.h — C ABI of the B200-native PillarAttn decode hot path.
 *
 * The reference (arXiv 2512.01278, `spardec`, /root/reference/pkg/src/spardec)
 * is pure Python/numpy: it has NO native plugin or FFI.  Its drop-in boundary
 * is the Python API; each entry point below replaces the arithmetic behind one
 * reference function, and the Python host package (paper_2512_01278_b200)
 * binds them with ctypes exactly where the reference calls that function:
 *
 *   sd_rope_kv_write      model.py:217-222 (_rotate) + model.py:271-287,326-331,
 *                         372-374 (KV rows pushed into the per-layer buffer)
 *   sd_attention          model.py:229-253 (_attend) as used by forward_full
 *                         (model.py:318-334, verify / prefill, with score
 *                         capture feeding selection.py:78-135) and by
 *                         forward_sparse (model.py:360-380, critical U fresh U self)
 *   sd_select_critical    engine.py:147-151 (_refresh_critical) =
 *                         selection.py:207-218 (importance_from_log) +
 *                         selection.py:167-183 (compute_budget) +
 *                         selection.py:186-204 (select_critical_tokens)
 *   sd_topk               selection.py:186-204 (select_critical_tokens)
 *   sd_argmax_rows        model.py:388-390 (greedy_token)
 *   sd_greedy_accept      engine.py:231-239 (verify_round accept loop + bonus)
 *   sd_step_prepare /     one unified iteration with device-resident request state
 *   sd_step_commit        (engine.py:196-260 per member; the delayed-verification
 *                         pipeline of scheduler.py:135-197, simulate.py:353-451)
 *
 * Conventions
 *   - Plain pointers and sizes only; every pointer is device memory unless
 *     stated.  The library never allocates: buffers and workspaces are owned
 *     by the caller (SURVEY.md §8b "Ownership").
 *   - Every call is asynchronous on the caller's cudaStream_t (passed as void*).
 *   - Return value: 0 = ok; < 0 = contract violation (message in
 *     sd_last_error(), thread-local); > 0 = CUDA error code.  The Python shim
 *     maps < 0 to ContractError and > 0 to RuntimeError (errors.py:8-37).
 */
#ifndef SPARDEC_B200_H
#define SPARDEC_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SD_ABI_VERSION 2

#define SD_DTYPE_F32 0
#define SD_DTYPE_BF16 1
#define SD_DTYPE_F64 2 /* sd_argmax_rows only */

/* Fields of one attention work item (int32 record of SD_ITEM_FIELDS). */
#define SD_ITEM_TABLE_ROW 0 /* block-table row of the request                      */
#define SD_ITEM_Q_ROW0 1    /* first query row in q/out                             */
#define SD_ITEM_NQ 2        /* query tokens in this item                            */
#define SD_ITEM_QPOS0 3     /* absolute position of query token 0                   */
#define SD_ITEM_CRIT_OFF 4  /* offset of this item's critical list in `crit`        */
#define SD_ITEM_CRIT_LEN 5  /* number of critical positions (all < DENSE_LO)        */
#define SD_ITEM_DENSE_LO 6  /* dense keys are [DENSE_LO, QPOS0 + NQ), causal        */
#define SD_ITEM_ACC_ROW 7   /* first score-accumulator row, -1 = no score capture   */
#define SD_ITEM_ACC_STEP 8  /* accumulator row step per query token (0 = sum rows)  */
#define SD_ITEM_FIELDS 12

/* One member of a unified iteration (int32 record of SD_PLAN_FIELDS), host -> device. */
#define SD_PLAN_SLOT 0  /* request slot (block-table row, state index)             */
#define SD_PLAN_KIND 1  /* SD_PLAN_DRAFT or SD_PLAN_VERIFY                          */
#define SD_PLAN_ROW0 2  /* first row of the member in the iteration's row batch     */
#define SD_PLAN_ROWS 3  /* 1 (draft) or round_target + 1 (verify)                   */
#define SD_PLAN_PHASE 4 /* draft step within the round (draft members)              */
#define SD_PLAN_ITEM 5  /* index into the draft / verify work items (and results)   */
#define SD_PLAN_FIELDS 6
#define SD_PLAN_DRAFT 0
#define SD_PLAN_VERIFY 1

/* Paged KV pool.  K and V: [layers][num_slots][kv_heads][head_dim] of dtype.
 * Logical position p of table row r lives in slot
 *   block_table[r * table_stride + (p >> page_shift)] << page_shift | (p & mask). */
typedef struct sd_paged_kv {
  void* k;
  void* v;
  int64_t layer_stride; /* elements between consecutive layers                 */
  int64_t num_slots;
  const int32_t* block_table;
  int32_t table_stride; /* pages per table row                                  */
  int32_t page_shift;   /* log2(tokens per page)                                */
  int32_t kv_heads;
  int32_t head_dim;
  int32_t dtype; /* SD_DTYPE_*                                                    */
  int32_t reserved;
} sd_paged_kv;

int32_t sd_abi_version(void);
/* Hash of the sources and build flags the library was compiled from. */
const char* sd_build_id(void);
const char* sd_last_error(void);
/* Number of kernels launched by this process through the library (evidence). */
int64_t sd_launch_count(void);

/* K5: RoPE (NeoX half split, base 1e4) of q and k at row_pos[r]; k and v are
 * written into the pool at (row_table[r], row_pos[r]) of `layer`; rotated q is
 * written to q_out [rows][q_heads][head_dim].  qkv row = [q | k | v]. */
int sd_rope_kv_write(const void* qkv, int64_t qkv_row_stride, int32_t rows,
                     const int32_t* row_table, const int32_t* row_pos,
                     const sd_paged_kv* kv, int32_t layer, int32_t q_heads,
                     void* q_out, void* stream);

/* K1 + K2: grouped-query attention of every item's query rows over its keys
 * (critical list, then dense causal range), two-phase exact softmax.
 *   q, out   : [rows][q_heads][head_dim] of kv->dtype
 *   lse      : [rows][q_heads] float or NULL
 *   items    : device int32 [num_items][SD_ITEM_FIELDS]
 *   crit     : device int32 critical positions (concatenated) or NULL
 *   acc      : uint64 fixed-point score accumulators (one unit = 2^-acc_shift);
 *              row a has acc_row_stride entries; for item query token t the row
 *              is ACC_ROW + t*ACC_STEP and
 *              acc[row][pos] += round(2^acc_shift * sum over the group's q heads
 *                                     of exp(s - lse))
 *              Integer addition makes the accumulated value independent of the
 *              order in which heads, CTAs and layers land (bitwise reproducible).
 *              Callers pick acc_shift so the largest possible entry (rows summed
 *              into it x layers x q_heads) stays below 2^62.
 *   planted  : device int32 sorted positions receiving +planted_bonus, or NULL
 *   max_keys, max_nq : host upper bounds over items (launch shaping)
 *   workspace: ZERO-FILLED device scratch of sd_attention_workspace_bytes() bytes;
 *              every call leaves it zero-filled again (reuse it across calls)
 *   flags    : bit0 = force the generic (FFMA) kernel
 * bf16 pools with head_dim 128 and GQA group 4 or 8 run the tcgen05 kernels for
 * items of up to 80 query rows (nq * group); other shapes run the generic kernel. */
int64_t sd_attention_workspace_bytes(int32_t num_items, int32_t max_keys, int32_t max_nq,
                                     int32_t q_heads, const sd_paged_kv* kv);
int sd_attention(const void* q, void* out, float* lse, const sd_paged_kv* kv, int32_t layer,
                 const int32_t* items, int32_t num_items, int32_t max_keys, int32_t max_nq,
                 const int32_t* crit, uint64_t* acc, int64_t acc_row_stride, int32_t acc_shift,
                 const int32_t* planted, int32_t num_planted, float planted_bonus,
                 int32_t q_heads, float scale, void* workspace, int64_t workspace_bytes,
                 int32_t flags, void* stream);

/* K3: per request r: importance[p] = 2^-acc_shift * sum_{t < n_rows[r]} acc[r][t][p]
 * (fp64, rows summed in order) for p < kv_len[r]; budget = max(1, min(ceil(s*n - 1e-9), n)) (n = 0 -> 1);
 * crit[r][:] = top-budget positions (value desc, ties to the lower index),
 * ascending; crit_len[r] = min(budget, kv_len[r]).
 * req_index (nullable): request r reads/writes row req_index[r] of acc,
 * importance, crit, crit_len and budget_out (n_rows / kv_len stay indexed by r). */
int sd_select_critical(const uint64_t* acc, int64_t acc_req_stride, int64_t acc_row_stride,
                       int32_t acc_shift, const int32_t* n_rows, const int32_t* kv_len, double sparsity,
                       int32_t num_requests, const int32_t* req_index,
                       double* importance, int64_t imp_stride,
                       int32_t* crit, int64_t crit_stride, int32_t* crit_len,
                       int32_t* budget_out, void* stream);

/* Plain top-k (selection.py:186-204) over float32 (dtype 0) or float64
 * (dtype 2) rows: values [num][stride], n[num], budget[num] -> out, out_len. */
int sd_topk(const void* values, int32_t value_dtype, int64_t stride, const int32_t* n,
            const int32_t* budget, int32_t num, int32_t* out, int64_t out_stride,
            int32_t* out_len, void* stream);

/* K4a: per-row argmax, ties to the lowest index.  logits [rows][row_stride] of
 * dtype F32, BF16 or F64 (fp64 rows are compared in fp64). */
int sd_argmax_rows(const void* logits, int32_t dtype, int64_t row_stride, int32_t rows,
                   int32_t vocab, int32_t* out, void* stream);

/* K4b: per verify member m: rows [row0[m], row0[m]+nrows[m]) hold the targets
 * of [pending, d_0 .. d_{n-2}]; tokens[] holds the verify INPUT tokens in the
 * same rows.  accepted[m] = longest prefix i with tokens[row0+1+i] ==
 * targets[row0+i]; bonus[m] = targets[row0 + accepted[m]]. */
int sd_greedy_accept(const int32_t* targets, const int32_t* tokens, const int32_t* row0,
                     const int32_t* nrows, int32_t num, int32_t* accepted, int32_t* bonus,
                     void* stream);

/* Unified iteration, device side (no host round trip between iterations).
 * Device state per request slot: n_kv[slot] committed KV rows, last_tok[slot] the
 * pending token (committed[-1]), drafted[slot][k] this round's drafts.
 * sd_step_prepare: from plan[n_members][SD_PLAN_FIELDS] writes the iteration's input
 *   tokens / row_table / row_pos, the verify work items v_items[...] (score capture into
 *   acc rows slot*(k+1)+j, zeroed here over [0, n_kv + rows)) and the draft work items
 *   d_items[...] (critical list at crit + slot*crit_cap, crit_len[slot], fresh tail from
 *   n_kv[slot]) (engine.py:196-231, model.py:360-365).
 * sd_step_commit (after sd_argmax_rows into targets[rows]): drafts store their target
 *   in drafted[slot][phase]; verifies apply the accept rule (engine.py:231-240), roll
 *   back n_kv += a + 1, set last_tok = bonus, write sel_rows/sel_kv/sel_slot[item] (the
 *   sd_select_critical inputs) and results[item][k+2] = {a, bonus, drafted[0..k-1]}. */
int sd_step_prepare(const int32_t* plan, int32_t n_members, int32_t k, int32_t crit_cap, const int32_t* n_kv,
                    const int32_t* last_tok, const int32_t* drafted, const int32_t* crit_len, int32_t* tokens,
                    int32_t* row_table, int32_t* row_pos, int32_t* v_items, int32_t* d_items, uint64_t* acc,
                    int64_t acc_row_stride, void* stream);
int sd_step_commit(const int32_t* plan, int32_t n_members, int32_t k, const int32_t* targets, int32_t* n_kv,
                   int32_t* last_tok, int32_t* drafted, int32_t* sel_rows, int32_t* sel_kv, int32_t* sel_slot,
                   int32_t* results, void* stream);

/* Glue (outside the attention hot path): out = x / sqrt(mean(x^2) + eps) per
 * row (model.py:225-226, RMSNorm without gain) cast to out_dtype.  x fp32. */
int sd_rmsnorm_cast(const float* x, int32_t rows, int32_t h, float eps, void* out, int32_t out_dtype,
                    void* stream);

/* One layer's bf16 weights (model.py:77-105), each stored out-major [out][in]
 * (nn.Linear layout; the reference's [in][out] matrix transposed). */
typedef struct sd_layer_weights {
  const void* w_qkv;   /* [(q_heads + 2 kv_heads) d][h]: rows of wq, then wk, then wv */
  const void* wo;      /* [h][h]   */
  const void* mlp_in;  /* [2h][h]  */
  const void* mlp_out; /* [h][2h]  */
} sd_layer_weights;

/* One sd_attention launch per layer (arguments as in sd_attention). */
typedef struct sd_attn_launch {
  const int32_t* items;
  int32_t num_items;
  int32_t max_keys;
  int32_t max_nq;
  int32_t acc_shift;
  const int32_t* crit;
  uint64_t* acc;
  int64_t acc_row_stride;
} sd_attn_launch;

/* The whole layer stack of one batched forward (model.py:290-342 for `rows` rows at
 * once; bf16 pools): per layer rmsnorm -> QKV GEMM -> K5 -> sd_attention for each launch
 * -> out-projection GEMM into the fp32 residual x -> rmsnorm -> MLP-in GEMM -> tanh ->
 * MLP-out GEMM into x.  GEMMs are cuBLAS (bf16 in, fp32 accumulate).  Buffers:
 * x fp32 [rows][h] (in/out); hn bf16 [rows][h]; qkv bf16 [rows][(q_heads+2kv_heads)d];
 * q, ctx bf16 [rows][q_heads][d]; hm bf16 [rows][2h].
 * Two launches (verify, draft) run concurrently per layer: the verify launch on a
 * high-priority stream, the draft launch on a low-priority one (forked from / joined
 * into `stream`), unless flags bit 0 is set or attn_events is given.
 * attn_events (nullable): cudaEvent_t pairs [layers][num_launches][2] recorded around
 * each attention launch (launches then run one after another).
 * flags bit 1: f3 fused verify + draft launch (sd_attention_pair); bit 3: the whole loop
 * is captured and launched as one CUDA graph (a cached executable updated in place each
 * call; falls back to direct launches when the capture is not possible). */
int sd_forward_layers(const sd_layer_weights* weights, int32_t layers, float* x, void* hn, void* qkv, void* q,
                      void* ctx, void* hm, int32_t rows, int32_t hidden, int32_t q_heads,
                      const int32_t* row_table, const int32_t* row_pos, const sd_paged_kv* kv,
                      const sd_attn_launch* launches, int32_t num_launches, const int32_t* planted,
                      int32_t num_planted, float planted_bonus, float scale, float eps, void* workspace,
                      int64_t workspace_bytes, void* const* attn_events, int32_t flags, void* stream);

/* f3: ONE launch for a layer's verify items (dense; score emission as in sd_attention) and
 * draft items (critical list + fresh tail, one query token, no score row): the verify
 * grid's CTAs claim the draft units (item, group of four kv heads) once their verify chunk
 * is done, so the drafts fill the verify launch's tail on chip.  Same buffers and work-item
 * format as two sd_attention calls; returns 1 without launching when the pair does not
 * qualify (bf16, head_dim 128, GQA 4/8, kv_heads % 4 == 0, <= 48 verify rows per item,
 * critical lists that stay TMEM-resident), 0 on success, else a CUDA error. */
int sd_attention_pair(const void* q, void* out, const sd_paged_kv* kv, int32_t layer, const sd_attn_launch* verify,
                      const sd_attn_launch* draft, const int32_t* planted, int32_t num_planted, float planted_bonus,
                      int32_t q_heads, float scale, void* stream);

/* One linear layer on the library's tuned cuBLASLt path (the LM head, model.py:339):
 * C[R][N] (+)= A[R][K] . W^T with A, W bf16 (W [N][K], nn.Linear layout), C fp32 when
 * c_f32 else bf16, beta 0 (overwrite) or 1 (accumulate). */
int sd_linear(const void* A, const void* W, void* C, int32_t R, int32_t N, int32_t K, int32_t c_f32, float beta,
              void* stream);

/* CUDA-graph path of sd_forward_layers on this thread and device: which 0 = executable
 * graphs instantiated, 1 = in-place updates (topology unchanged since the last call). */
int64_t sd_forward_graph_stats(int32_t which);

/* Workspace sd_forward_layers needs: the attention launches' (sd_attention_workspace_bytes,
 * max over the launches) plus a RoPE cos/sin table of `rows` rows kept at its end. */
int64_t sd_forward_workspace_bytes(int32_t rows, int32_t head_dim, int64_t attention_bytes);

#ifdef __cplusplus
}
#endif

#endif /* SPARDEC_B200_H */
