// Instantiations of the tcgen05 verify kernel for GQA group 8 (split from attn_umma.cu so
// the two groups compile in parallel).
#include "attn_umma.cuh"

namespace sd {
namespace umma_attn {

int launch_verify_g8(const Params& prm, int NR, int C, int num_items, int kv_heads, cudaStream_t stream) {
  switch (NR) {
    case 8: return launch_verify<8, 8, 2, 256>(prm, C, num_items, kv_heads, stream);
    case 16: return launch_verify<8, 16, 2, 256>(prm, C, num_items, kv_heads, stream);
    case 24: return launch_verify<8, 24, 2, 256>(prm, C, num_items, kv_heads, stream);
    case 32: return launch_verify<8, 32, 2, 256>(prm, C, num_items, kv_heads, stream);
    case 40: return launch_verify<8, 40, 2, 256>(prm, C, num_items, kv_heads, stream);
    case 48: return launch_verify<8, 48, 2, 256>(prm, C, num_items, kv_heads, stream);
    case 56: return launch_verify<8, 56, 4, 512>(prm, C, num_items, kv_heads, stream);
    case 64: return launch_verify<8, 64, 4, 512>(prm, C, num_items, kv_heads, stream);
    case 72: return launch_verify<8, 72, 4, 512>(prm, C, num_items, kv_heads, stream);
    case 80: return launch_verify<8, 80, 4, 512>(prm, C, num_items, kv_heads, stream);
    default: break;
  }
  set_error("sd_attention (umma): no verify kernel for NR = " + std::to_string(NR));
  return -1;
}

}  // namespace umma_attn
}  // namespace sd
