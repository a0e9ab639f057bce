// K2 tcgen05/TMA variant (bf16, dh = 128) — placeholder until the kernel lands.
#include "common.cuh"

namespace propd {

int attention_tc_bf16(int, int, int, int, int, int, const void*, int, const void*, const void*, const int32_t*,
                      const int32_t*, const int32_t*, const int32_t*, const uint64_t*, int, int, void*, int, void*,
                      int64_t, cudaStream_t, bool* handled) {
  *handled = false;
  return 0;
}

}  // namespace propd
