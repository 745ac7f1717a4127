// C-ABI surface: error state, launch accounting, attention dispatch.
#include <atomic>
#include <string>

#include "common.cuh"

namespace sd {

static thread_local std::string g_last_error;
static std::atomic<long long> g_launches{0};

void set_error(const std::string& msg) { g_last_error = msg; }
void count_launch(int n) { g_launches.fetch_add(n, std::memory_order_relaxed); }

int64_t generic_ws_bytes(int num_items, int max_keys, int max_rows, int kv_heads);
int launch_attn_generic(const void* q, void* out, float* lse, const sd_paged_kv* kvp, int layer,
                        const int32_t* items, int num_items, int max_keys, int max_nq, const int32_t* crit,
                        unsigned long long* acc, int64_t acc_stride, int acc_shift, const int32_t* planted,
                        int n_planted, float bonus, int q_heads, float scale, void* ws, int64_t ws_bytes,
                        cudaStream_t stream);
bool umma_supported(const sd_paged_kv* kvp, int max_nq, int q_heads);
int launch_attn_umma(const void* q, void* out, float* lse, const sd_paged_kv* kvp, int layer, const int32_t* items,
                     int num_items, int max_keys, int max_nq, const int32_t* crit, unsigned long long* acc,
                     int64_t acc_stride, int acc_shift, const int32_t* planted, int n_planted, float bonus,
                     int q_heads, float scale, void* ws, int64_t ws_bytes, cudaStream_t stream, bool* handled);

}  // namespace sd

#ifndef SD_BUILD_ID
#define SD_BUILD_ID "unknown"
#endif

extern "C" int32_t sd_abi_version(void) { return SD_ABI_VERSION; }
// hash of the sources and flags this library was compiled from (csrc/build.py source_stamp)
extern "C" const char* sd_build_id(void) { return SD_BUILD_ID; }
extern "C" const char* sd_last_error(void) { return sd::g_last_error.c_str(); }
extern "C" int64_t sd_launch_count(void) { return sd::g_launches.load(); }

extern "C" int64_t sd_attention_workspace_bytes(int32_t num_items, int32_t max_keys, int32_t max_nq,
                                                int32_t q_heads, const sd_paged_kv* kv) {
  if (kv == nullptr || kv->kv_heads <= 0) return 0;
  if (sd::umma_supported(kv, max_nq, q_heads)) return 0;  // tcgen05: partials meet in DSMEM
  const int G = q_heads / kv->kv_heads;
  return sd::generic_ws_bytes(num_items, max_keys, max_nq * G, kv->kv_heads);
}

// One dispatch rule, no fallback chain: the tcgen05 kernels (attn_umma*.cu) take every bf16
// shape they cover (head_dim 128, GQA 4/8, <= 80 query rows per item); the generic FFMA
// kernel takes the rest (fp32 parity mode, other head dims / groups) and flag bit 0.
extern "C" int sd_attention(const void* q, void* out, float* lse, const sd_paged_kv* kv, int32_t layer,
                            const int32_t* items, int32_t num_items, int32_t max_keys, int32_t max_nq,
                            const int32_t* crit, uint64_t* acc, int64_t acc_row_stride, int32_t acc_shift,
                            const int32_t* planted, int32_t num_planted, float planted_bonus, int32_t q_heads,
                            float scale, void* workspace, int64_t workspace_bytes, int32_t flags, void* stream) {
  SD_REQUIRE(kv != nullptr && q != nullptr && out != nullptr && items != nullptr, "sd_attention: null pointer");
  SD_REQUIRE(kv->kv_heads > 0 && q_heads % kv->kv_heads == 0, "sd_attention: kv_heads must divide q_heads");
  SD_REQUIRE(kv->dtype == SD_DTYPE_F32 || kv->dtype == SD_DTYPE_BF16, "sd_attention: unsupported dtype");
  SD_REQUIRE(kv->page_shift >= 0 && kv->page_shift < 16, "sd_attention: bad page_shift");
  SD_REQUIRE(max_nq >= 1 && max_keys >= 1, "sd_attention: max_nq and max_keys must be positive");
  SD_REQUIRE(num_planted == 0 || planted != nullptr, "sd_attention: planted list missing");
  SD_REQUIRE(acc == nullptr || (acc_shift >= 0 && acc_shift <= 62), "sd_attention: acc_shift must be in [0, 62]");
  if (num_items == 0) return 0;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  unsigned long long* a = reinterpret_cast<unsigned long long*>(acc);
  if (!(flags & 1)) {
    bool handled = false;
    const int rc = sd::launch_attn_umma(q, out, lse, kv, layer, items, num_items, max_keys, max_nq, crit, a,
                                        acc_row_stride, acc_shift, planted, num_planted, planted_bonus, q_heads,
                                        scale, workspace, workspace_bytes, s, &handled);
    if (handled || rc != 0) return rc;
  }
  return sd::launch_attn_generic(q, out, lse, kv, layer, items, num_items, max_keys, max_nq, crit, a,
                                 acc_row_stride, acc_shift, planted, num_planted, planted_bonus, q_heads, scale,
                                 workspace, workspace_bytes, s);
}
