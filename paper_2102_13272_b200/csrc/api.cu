// api.cu -- device-side half of the C ABI: argument checks, workspace carving
// and the launch sequence of each path.  Every path is our own kernels; there
// is no CPU or library fallback (a missing kernel returns NW_ERR_UNSUPPORTED).
#include "nw_internal.h"

using namespace nw;

namespace {
inline bool aligned16(const void *ptr) { return (reinterpret_cast<uintptr_t>(ptr) & 15u) == 0; }
}  // namespace

extern "C" {

nw_status_t nw_transform_filter(nw_plan_t p, const void *w, void *U, nw_stream_t stream) {
  if (!p || !w || !U) return NW_ERR_INVALID;
  nw_status_t st = finalize(p);
  if (st != NW_OK) return st;
  if (!aligned16(U)) return NW_ERR_INVALID;
  Geometry g = make_geometry(p, 1, 64, 64);
  return launch_filter_transform(p, g, w, U, reinterpret_cast<cudaStream_t>(stream));
}

nw_status_t nw_conv_forward(nw_plan_t p, const void *x, const void *U, void *y, int N, int H, int W, void *ws,
                            size_t ws_bytes, nw_stream_t stream) {
  if (!p || !x || !U || !y || N < 1 || H < 1 || W < 1) return NW_ERR_INVALID;
  nw_status_t st = finalize(p);
  if (st != NW_OK) return st;
  if (!aligned16(x) || !aligned16(U) || !aligned16(y) || !aligned16(ws)) return NW_ERR_INVALID;
  Geometry g = make_geometry(p, N, H, W);
  if (g.Ho < 1 || g.Wo < 1) return NW_ERR_INVALID;
  const size_t vb = v_bytes(p, g), mb = m_bytes(p, g);
  if (!ws || ws_bytes < vb + mb) return NW_ERR_WORKSPACE;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  char *base = static_cast<char *>(ws);
  void *V = base;
  float *M = reinterpret_cast<float *>(base + vb);
  if ((st = launch_input_transform(p, g, x, V, s)) != NW_OK) return st;
  if (p->math == NW_MATH_FP32_SIMT)
    st = launch_gemm_simt(p, g, static_cast<const float *>(V), static_cast<const float *>(U), M, s);
  else
    st = launch_gemm_tc(p, g, V, U, M, s);
  if (st != NW_OK) return st;
  return launch_output_transform(p, g, M, y, s);
}

}  // extern "C"
