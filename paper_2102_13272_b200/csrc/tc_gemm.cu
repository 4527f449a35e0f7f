// tc_gemm.cu -- tcgen05 contraction (placeholder until the kernel lands).
#include "nw_internal.h"

namespace nw {
nw_status_t launch_gemm_tc(const nw_plan_st *, const Geometry &, const void *, const void *, float *, cudaStream_t) {
  return NW_ERR_UNSUPPORTED;
}
}  // namespace nw
