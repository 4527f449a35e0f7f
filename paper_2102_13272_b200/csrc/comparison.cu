// comparison.cu -- OLA-Winograd and direct implicit-GEMM comparison paths (placeholder).
#include "nw_internal.h"

extern "C" {
nw_status_t nw_workspace_size_ola(nw_plan_t p, int N, int H, int W, size_t *bytes) {
  (void)p; (void)N; (void)H; (void)W; (void)bytes;
  return NW_ERR_UNSUPPORTED;
}
nw_status_t nw_workspace_size_direct(nw_plan_t p, int N, int H, int W, size_t *bytes) {
  (void)p; (void)N; (void)H; (void)W; (void)bytes;
  return NW_ERR_UNSUPPORTED;
}
nw_status_t nw_conv_ola(nw_plan_t, const void *, const void *, void *, int, int, int, void *, size_t, nw_stream_t) {
  return NW_ERR_UNSUPPORTED;
}
nw_status_t nw_conv_direct(nw_plan_t, const void *, const void *, void *, int, int, int, void *, size_t,
                           nw_stream_t) {
  return NW_ERR_UNSUPPORTED;
}
}
