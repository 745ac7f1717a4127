// Instantiations of the tcgen05 verify kernel for GQA group 8 (split from attn_umma.cu so
// the two groups compile in parallel).
#include "attn_umma.cuh"

namespace sd {
namespace umma_attn {

#define SD_VERIFY_SHAPES(X) \
  X(8, 2, 256) X(16, 2, 256) X(24, 2, 256) X(32, 2, 256) X(40, 2, 256) X(48, 2, 256) \
  X(56, 4, 512) X(64, 4, 512) X(72, 4, 512) X(80, 4, 512)

int launch_verify_g8(const Params& prm, int NR, int C, int num_items, int kv_heads, cudaStream_t stream) {
  switch (NR) {
#define X(nr, ns, tc) \
  case nr: return launch_verify<8, nr, ns, tc>(prm, C, num_items, kv_heads, stream);
    SD_VERIFY_SHAPES(X)
#undef X
    default: break;
  }
  set_error("sd_attention (umma): no verify kernel for NR = " + std::to_string(NR));
  return -1;
}

int launch_fused_g8(const Params& pv, const Params& pd, const FusedCtl& fc, int NR, int C, int num_items, int kv_heads,
                    int smem, cudaStream_t stream) {
  switch (NR) {
#define X(nr) \
  case nr: return launch_fused<8, nr, 2, 256>(pv, pd, fc, C, num_items, kv_heads, smem, stream);
    X(8) X(16) X(24) X(32) X(40) X(48)
#undef X
    default: break;
  }
  return -1;
}

int verify_slots_g8(int NR, int C, int smem) {
  switch (NR) {
#define X(nr, ns, tc) \
  case nr: return verify_slots<8, nr, ns, tc>(C, smem);
    SD_VERIFY_SHAPES(X)
#undef X
    default: break;
  }
  return 0;
}

}  // namespace umma_attn
}  // namespace sd
