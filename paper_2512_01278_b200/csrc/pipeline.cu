// Device-resident request state for the unified draft/verify iteration, so the host can
// enqueue iteration i+1 before it has read iteration i's accept/reject results (SURVEY.md
// §8 f2; the delayed-verification pipeline of scheduler.py:135-197 / simulate.py:353-451).
//
// Per request slot the device keeps
//   n_kv[slot]          committed KV rows (prompt + committed - 1: the pending token's KV is
//                       written by the next forward, engine.py:98-100)
//   last_tok[slot]      committed[-1], the pending token
//   drafted[slot][k]    this round's drafted tokens
// and each iteration is
//   sd_step_prepare   plan (host: slot, kind, row0, rows, phase, item) -> tokens, positions,
//                     block-table rows and the K1 / K2 work items, from the device state;
//                     zeroes the verify members' score-accumulator rows
//   ... forward (sd_forward_layers), LM head, sd_argmax_rows ...
//   sd_step_commit    drafts: drafted[slot][phase] = target; verifies: accept rule
//                     (engine.py:231-240: a = longest prefix with drafted[i] == target[i],
//                     bonus = target[a]), KV rollback n_kv += a + 1, last_tok = bonus, the K3
//                     inputs (surviving rows a + 1, kv length) and the host result record
//                     (a, bonus, drafted[0 .. rows-2]) for the delayed host-side processing.
#include "common.cuh"

namespace sd {

__global__ void step_prepare_kernel(const int32_t* __restrict__ plan, int n_members, int k, int crit_cap,
                                    const int32_t* __restrict__ n_kv, const int32_t* __restrict__ last_tok,
                                    const int32_t* __restrict__ drafted, const int32_t* __restrict__ crit_len,
                                    int32_t* __restrict__ tokens, int32_t* __restrict__ row_table,
                                    int32_t* __restrict__ row_pos, int32_t* __restrict__ v_items,
                                    int32_t* __restrict__ d_items, unsigned long long* __restrict__ acc,
                                    int64_t acc_row_stride) {
  const int m = blockIdx.x;
  const int32_t* pl = plan + (int64_t)m * SD_PLAN_FIELDS;
  const int slot = pl[SD_PLAN_SLOT], kind = pl[SD_PLAN_KIND], row0 = pl[SD_PLAN_ROW0];
  const int rows = pl[SD_PLAN_ROWS], phase = pl[SD_PLAN_PHASE], item = pl[SD_PLAN_ITEM];
  const int n0 = n_kv[slot];
  const int32_t* dr = drafted + (int64_t)slot * k;
  if (kind == SD_PLAN_DRAFT) {
    if (threadIdx.x == 0) {
      // the draft at step `phase` of the round: token drafted[-1] (or the pending token),
      // position n0 + phase, attends to critical U [n0, n0 + phase] (model.py:360-365)
      tokens[row0] = phase == 0 ? last_tok[slot] : dr[phase - 1];
      row_table[row0] = slot;
      row_pos[row0] = n0 + phase;
      int32_t* it = d_items + (int64_t)item * SD_ITEM_FIELDS;
      it[SD_ITEM_TABLE_ROW] = slot;
      it[SD_ITEM_Q_ROW0] = row0;
      it[SD_ITEM_NQ] = 1;
      it[SD_ITEM_QPOS0] = n0 + phase;
      it[SD_ITEM_CRIT_OFF] = slot * crit_cap;
      it[SD_ITEM_CRIT_LEN] = crit_len[slot];
      it[SD_ITEM_DENSE_LO] = n0;
      it[SD_ITEM_ACC_ROW] = -1;
      it[SD_ITEM_ACC_STEP] = 0;
    }
    return;
  }
  // verify: rows [committed[-1], drafted[0 .. rows-2]] at n0 .. n0 + rows - 1 (engine.py:231)
  for (int j = threadIdx.x; j < rows; j += blockDim.x) {
    tokens[row0 + j] = j == 0 ? last_tok[slot] : dr[j - 1];
    row_table[row0 + j] = slot;
    row_pos[row0 + j] = n0 + j;
  }
  if (threadIdx.x == 0) {
    int32_t* it = v_items + (int64_t)item * SD_ITEM_FIELDS;
    it[SD_ITEM_TABLE_ROW] = slot;
    it[SD_ITEM_Q_ROW0] = row0;
    it[SD_ITEM_NQ] = rows;
    it[SD_ITEM_QPOS0] = n0;
    it[SD_ITEM_CRIT_OFF] = 0;
    it[SD_ITEM_CRIT_LEN] = 0;
    it[SD_ITEM_DENSE_LO] = 0;
    it[SD_ITEM_ACC_ROW] = slot * (k + 1);
    it[SD_ITEM_ACC_STEP] = 1;
  }
  // the verify kernel accumulates scores into acc[slot*(k+1) + j][0 .. n0 + rows): zero them
  const int width = n0 + rows;
  for (int j = 0; j < rows; ++j) {
    unsigned long long* a = acc + (int64_t)(slot * (k + 1) + j) * acc_row_stride;
    for (int p = threadIdx.x; p < width; p += blockDim.x) a[p] = 0ull;
  }
}

__global__ void step_commit_kernel(const int32_t* __restrict__ plan, int n_members, int k,
                                   const int32_t* __restrict__ targets, int32_t* __restrict__ n_kv,
                                   int32_t* __restrict__ last_tok, int32_t* __restrict__ drafted,
                                   int32_t* __restrict__ sel_rows, int32_t* __restrict__ sel_kv,
                                   int32_t* __restrict__ sel_slot, int32_t* __restrict__ results) {
  const int m = blockIdx.x * blockDim.x + threadIdx.x;
  if (m >= n_members) return;
  const int32_t* pl = plan + (int64_t)m * SD_PLAN_FIELDS;
  const int slot = pl[SD_PLAN_SLOT], kind = pl[SD_PLAN_KIND], row0 = pl[SD_PLAN_ROW0];
  const int rows = pl[SD_PLAN_ROWS], phase = pl[SD_PLAN_PHASE], item = pl[SD_PLAN_ITEM];
  int32_t* dr = drafted + (int64_t)slot * k;
  if (kind == SD_PLAN_DRAFT) {
    if (phase < k) dr[phase] = targets[row0];
    return;
  }
  int a = 0;
  while (a < rows - 1 && dr[a] == targets[row0 + a]) ++a;
  const int bonus = targets[row0 + a];
  int32_t* res = results + (int64_t)item * (k + 2);
  res[0] = a;
  res[1] = bonus;
  for (int i = 0; i < k; ++i) res[2 + i] = i < rows - 1 ? dr[i] : -1;
  const int n1 = n_kv[slot] + a + 1;  // KV rollback: rows past n0 + a are dead (engine.py:240)
  n_kv[slot] = n1;
  last_tok[slot] = bonus;
  sel_rows[item] = a + 1;  // importance over the surviving rows 0..a (engine.py:258)
  sel_kv[item] = n1;
  sel_slot[item] = slot;
}

}  // namespace sd

extern "C" int sd_step_prepare(const int32_t* plan, int32_t n_members, int32_t k, int32_t crit_cap,
                               const int32_t* n_kv, const int32_t* last_tok, const int32_t* drafted,
                               const int32_t* crit_len, int32_t* tokens, int32_t* row_table, int32_t* row_pos,
                               int32_t* v_items, int32_t* d_items, uint64_t* acc, int64_t acc_row_stride,
                               void* stream) {
  SD_REQUIRE(n_members >= 0 && k >= 1, "sd_step_prepare: bad sizes");
  if (n_members == 0) return 0;
  SD_REQUIRE(plan && n_kv && last_tok && drafted && crit_len && tokens && row_table && row_pos,
             "sd_step_prepare: null pointer");
  sd::step_prepare_kernel<<<n_members, 128, 0, static_cast<cudaStream_t>(stream)>>>(
      plan, n_members, k, crit_cap, n_kv, last_tok, drafted, crit_len, tokens, row_table, row_pos, v_items, d_items,
      reinterpret_cast<unsigned long long*>(acc), acc_row_stride);
  sd::count_launch();
  SD_CUDA_RETURN();
}

extern "C" int sd_step_commit(const int32_t* plan, int32_t n_members, int32_t k, const int32_t* targets,
                              int32_t* n_kv, int32_t* last_tok, int32_t* drafted, int32_t* sel_rows, int32_t* sel_kv,
                              int32_t* sel_slot, int32_t* results, void* stream) {
  SD_REQUIRE(n_members >= 0 && k >= 1, "sd_step_commit: bad sizes");
  if (n_members == 0) return 0;
  SD_REQUIRE(plan && targets && n_kv && last_tok && drafted && sel_rows && sel_kv && sel_slot && results,
             "sd_step_commit: null pointer");
  sd::step_commit_kernel<<<(n_members + 127) / 128, 128, 0, static_cast<cudaStream_t>(stream)>>>(
      plan, n_members, k, targets, n_kv, last_tok, drafted, sel_rows, sel_kv, sel_slot, results);
  sd::count_launch();
  SD_CUDA_RETURN();
}
