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

extern "C" {

nw_status_t nw_workspace_size_host(nw_plan_t p, int N, int H, int W, size_t *bytes) {
  size_t b = 0;
  nw_status_t st = nw_workspace_size(p, N, H, W, &b);
  if (st != NW_OK) return st;
  Geometry g = make_geometry(p, N, H, W);
  const size_t es = (p->dtype == NW_DTYPE_BF16) ? 2 : 4;
  const size_t xb = (size_t)round_up((long long)N * p->Cin * H * W * es, 256);
  const size_t yb = (size_t)round_up((long long)N * p->Cout * g.Ho * g.Wo * es, 256);
  *bytes = b + xb + yb;
  return NW_OK;
}

nw_status_t nw_conv_forward_host(nw_plan_t p, const void *x_host, const void *U, void *y_host, int N, int H, int W,
                                 void *ws, size_t ws_bytes, nw_stream_t stream) {
  if (!p || !x_host || !y_host || !U || N < 1 || H < 1 || W < 1) return NW_ERR_INVALID;
  size_t need = 0;
  nw_status_t st = nw_workspace_size_host(p, N, H, W, &need);
  if (st != NW_OK) return st;
  if (!ws || ws_bytes < need) return NW_ERR_WORKSPACE;
  Geometry g = make_geometry(p, N, H, W);
  const size_t es = (p->dtype == NW_DTYPE_BF16) ? 2 : 4;
  const size_t xbytes = (size_t)N * p->Cin * H * W * es;
  const size_t ybytes = (size_t)N * p->Cout * g.Ho * g.Wo * es;
  const size_t fw = v_bytes(p, g) + m_bytes(p, g);
  char *base = static_cast<char *>(ws);
  char *xd = base + fw;
  char *yd = xd + (size_t)round_up((long long)xbytes, 256);
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  if (cudaMemcpyAsync(xd, x_host, xbytes, cudaMemcpyHostToDevice, s) != cudaSuccess) return NW_ERR_CUDA;
  st = nw_conv_forward(p, xd, U, yd, N, H, W, ws, fw, stream);
  if (st != NW_OK) return st;
  if (cudaMemcpyAsync(y_host, yd, ybytes, cudaMemcpyDeviceToHost, s) != cudaSuccess) return NW_ERR_CUDA;
  return NW_OK;
}

}  // extern "C"
