// tc.cu -- tcgen05 (TMEM accumulator) path of the chunked negative contraction. Filled in by the TC milestone.
#include "kge_internal.h"

namespace kge {

bool tc_supported(const kge_handle* h) {
  (void)h;
  return false;
}

cudaError_t launch_tc_neg(kge_handle* h, const Slot& s) {
  (void)h;
  (void)s;
  return cudaErrorNotSupported;
}

}  // namespace kge
