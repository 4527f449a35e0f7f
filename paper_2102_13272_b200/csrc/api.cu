// api.cu -- device-side half of the C ABI: argument checks, workspace carving
// and the launch sequence of each path.  Every path is our own kernels; there
// is no CPU or library fallback (a missing kernel returns NW_ERR_UNSUPPORTED).
#include <cstdlib>
#include <vector>

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

}  // extern "C"

namespace nw {

// grow a plan's event pool to n events (caller holds the pool's mutex)
static bool ensure_events(std::vector<cudaEvent_t> &pool, size_t n) {
  while (pool.size() < n) {
    cudaEvent_t e = nullptr;
    if (cudaEventCreateWithFlags(&e, cudaEventDisableTiming) != cudaSuccess) return false;
    pool.push_back(e);
  }
  return true;
}

static int env_int(const char *name, int dflt) {
  const char *v = getenv(name);
  return (v && *v) ? atoi(v) : dflt;
}

// Chunk pipeline of the forward pass: the batch is cut into k chunks; chunk c's
// input transform, contraction and output transform run on three streams, so
// the CUDA-core transforms of one chunk overlap the HBM-bound tensor-core
// contraction of the next.  V / M are double buffered.
int forward_chunks(const nw_plan_st *p, int N, int H, int W) {
  int k = p->pipe_chunks >= 0 ? p->pipe_chunks : env_int("NW_PIPE_CHUNKS", 1);
  if (k > N) k = N;
  if (k < 1) k = 1;
  Geometry g = make_geometry(p, 1, H, W);
  const size_t es = (p->dtype == NW_DTYPE_BF16) ? 2 : 4;
  // chunk pointers must stay 16-byte aligned
  if (((size_t)p->Cin * H * W * es) % 16 || ((size_t)p->Cout * g.Ho * g.Wo * es) % 16) k = 1;
  return k;
}

// completion counters of the streamed pipeline: two per 128-slice block
static size_t sync_bytes(const Geometry &g) { return (size_t)round_up(2 * (g.T_pad / 128) * 4, 256); }

size_t forward_ws_bytes(const nw_plan_st *p, int N, int H, int W) {
  const int k = forward_chunks(p, N, H, W);
  const int nc = (N + k - 1) / k;
  Geometry g = make_geometry(p, nc, H, W);
  return (size_t)(k > 1 ? 2 : 1) * (v_bytes(p, g) + m_bytes(p, g)) + sync_bytes(g);
}

// Streamed pipeline (NW_STREAM=1): the input transform and the fused contraction run at the
// same time on disjoint SM sets, connected by per-128-slice-block completion counters, so the
// contraction reads each block's V from L2 shortly after it is written instead of from HBM
// (L2-resident reads measured at ~19 TB/s against 7 TB/s from HBM, tools/l2_bw2.cu).  The
// input transform never waits on the contraction, so the pair cannot deadlock as long as the
// input transform's CTAs are resident (launched first, on fewer SMs than the GPU has).
static int stream_mode() {  // NW_STREAM: 0 off, 1 input || contraction, 2 contraction || output, 3 all three
  static const int m = env_int("NW_STREAM", 0);
  return m;
}

static nw_status_t forward_streamed(nw_plan_st *p, const Geometry &g, const void *x, const void *U, void *y,
                                    void *V, float *M, int *sync, cudaStream_t s, bool *done) {
  *done = false;
  const int mode = stream_mode();
  int sms = 148, dev = 0;
  if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  static const int k_it = env_int("NW_STREAM_IT", 64), k_ot = env_int("NW_STREAM_OT", 48);
  const bool s_in = mode == 1 || mode == 3, s_out = mode == 2 || mode == 3;
  const int k1 = s_in ? k_it : 0, k3 = s_out ? k_ot : 0;
  if ((s_in && k1 < 1) || (s_out && k3 < 1) || k1 + k3 >= sms) return NW_OK;
  const long long nmb = g.T_pad / 128;
  Geometry gs = g;
  gs.sync = s_in ? sync : nullptr;
  gs.sync2 = s_out ? sync + nmb : nullptr;
  gs.it_ctas = k1;
  gs.ot_ctas = k3;
  gs.gemm_ctas = sms - k1 - k3;
  std::lock_guard<std::mutex> lk(p->pipe_mu);
  for (int i = 0; i < 3; ++i)
    if (!p->s_pipe[i] && cudaStreamCreateWithFlags(&p->s_pipe[i], cudaStreamNonBlocking) != cudaSuccess)
      return NW_ERR_CUDA;
  if (!ensure_events(p->ev_pipe, 4)) return NW_ERR_CUDA;
  cudaStream_t sa = p->s_pipe[0], sb = p->s_pipe[1], sc = p->s_pipe[2];
  cudaEvent_t e0 = p->ev_pipe[0], ea = p->ev_pipe[1], eb = p->ev_pipe[2], ec = p->ev_pipe[3];
  nw_status_t st;
  if (!s_in) {  // the input transform alone on every SM, before the concurrent pair
    Geometry gi = g;
    if ((st = launch_input_transform(p, gi, x, V, s)) != NW_OK) return st;
  }
  if (cudaMemsetAsync(sync, 0, (size_t)nmb * 8, s) != cudaSuccess) return NW_ERR_CUDA;
  if (cudaEventRecord(e0, s) != cudaSuccess) return NW_ERR_CUDA;
  for (cudaStream_t t : {sa, sb, sc})
    if (cudaStreamWaitEvent(t, e0, 0) != cudaSuccess) return NW_ERR_CUDA;
  // launch order = dependency order: a consumer's producer is dispatched first
  if (s_in) {
    st = launch_input_transform(p, gs, x, V, sa);
    if (st == NW_ERR_UNSUPPORTED) return NW_OK;  // no signalling input transform for this layer
    if (st != NW_OK) return st;
  }
  if ((st = launch_gemm_tc_fused(p, gs, V, U, M, sb)) != NW_OK) return st;
  if (s_out) {
    if ((st = launch_output_transform_pre(p, gs, M, y, sc)) != NW_OK) return st;
  }
  if (cudaEventRecord(ea, sa) != cudaSuccess || cudaEventRecord(eb, sb) != cudaSuccess ||
      cudaEventRecord(ec, sc) != cudaSuccess)
    return NW_ERR_CUDA;
  for (cudaEvent_t e : {ea, eb, ec})
    if (cudaStreamWaitEvent(s, e, 0) != cudaSuccess) return NW_ERR_CUDA;
  *done = true;
  return s_out ? NW_OK : launch_output_transform_pre(p, g, M, y, s);
}

static nw_status_t forward_one(const nw_plan_st *p, const Geometry &g, const void *x, const void *U, void *y, void *V,
                               float *M, cudaStream_t si, cudaStream_t sg, cudaStream_t so, cudaEvent_t e_in,
                               cudaEvent_t e_gemm, int *sync = nullptr) {
  nw_status_t st;
  if (sync && stream_mode() && si == so && sg == so && gemm_fused_eligible(p, g) && !p->depthwise &&
      !fused_c1_eligible(p, g) && !fused_co_eligible(p, g)) {
    bool done = false;
    // the plan's stream / event caches are mutable state of an otherwise const plan
    if ((st = forward_streamed(const_cast<nw_plan_st *>(p), g, x, U, y, V, M, sync, si, &done)) != NW_OK) return st;
    if (done) return NW_OK;
  }
  if (fused_c1_eligible(p, g)) {  // one input channel: V and M never leave the SM
    if ((st = launch_fused_c1(p, g, x, U, y, V, v_bytes(p, g), si)) != NW_OK) return st;
    if (si != so) {
      if (cudaEventRecord(e_in, si) != cudaSuccess || cudaStreamWaitEvent(so, e_in, 0) != cudaSuccess)
        return NW_ERR_CUDA;
    }
    return NW_OK;
  }
  if (fused_co_eligible(p, g)) {  // Cout_e <= 4: V and M never leave the SM
    if ((st = launch_fused_co(p, g, x, U, y, V, si)) != NW_OK) return st;
    if (si != so) {
      if (cudaEventRecord(e_in, si) != cudaSuccess || cudaStreamWaitEvent(so, e_in, 0) != cudaSuccess)
        return NW_ERR_CUDA;
    }
    return NW_OK;
  }
  if ((st = launch_input_transform(p, g, x, V, si)) != NW_OK) return st;
  if (p->depthwise) {  // no channel contraction: per-channel product, then the plain output transform
    if ((st = launch_depthwise_product(p, g, V, static_cast<const float *>(U), M, si)) != NW_OK) return st;
    if (si != so) {
      if (cudaEventRecord(e_in, si) != cudaSuccess || cudaStreamWaitEvent(so, e_in, 0) != cudaSuccess)
        return NW_ERR_CUDA;
    }
    return launch_output_transform(p, g, M, y, so);
  }
  if (si != sg) {
    if (cudaEventRecord(e_in, si) != cudaSuccess || cudaStreamWaitEvent(sg, e_in, 0) != cudaSuccess) return NW_ERR_CUDA;
  }
  const int flevel = gemm_fused_level(p, g);  // inner output level(s) in the contraction epilogue
  const bool fused = flevel > 0;
  if (p->math == NW_MATH_FP32_SIMT)
    st = launch_gemm_simt(p, g, static_cast<const float *>(V), static_cast<const float *>(U), M, sg);
  else if (flevel == 2)
    st = launch_gemm_tc_fused2(p, g, V, U, M, sg);
  else if (fused && gemm_fused_wide(p, g))
    st = launch_gemm_tc_fused1c(p, g, V, U, M, sg);
  else if (fused)
    st = launch_gemm_tc_fused(p, g, V, U, M, sg);
  else
    st = launch_gemm_tc(p, g, V, U, M, sg);
  if (st != NW_OK) return st;
  if (sg != so) {
    if (cudaEventRecord(e_gemm, sg) != cudaSuccess || cudaStreamWaitEvent(so, e_gemm, 0) != cudaSuccess)
      return NW_ERR_CUDA;
  }
  if (flevel == 2) return launch_output_transform_pre2(p, g, M, y, so);
  return fused ? launch_output_transform_pre(p, g, M, y, so) : launch_output_transform(p, g, M, y, so);
}

}  // namespace nw

extern "C" {

nw_status_t nw_conv_forward(nw_plan_t p, const void *x, const void *U, void *y, int N, int H, int W, void *ws,
                            size_t ws_bytes, nw_stream_t stream) {
  if (!p || !x || !U || !y || N < 1 || H < 1 || W < 1) return NW_ERR_INVALID;
  nw_status_t st = finalize(p);
  if (st != NW_OK) return st;
  if (!aligned16(x) || !aligned16(U) || !aligned16(y) || !aligned16(ws)) return NW_ERR_INVALID;
  Geometry gfull = make_geometry(p, N, H, W);
  if (gfull.Ho < 1 || gfull.Wo < 1) return NW_ERR_INVALID;
  if (!ws || ws_bytes < forward_ws_bytes(p, N, H, W)) return NW_ERR_WORKSPACE;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  const int k = forward_chunks(p, N, H, W);
  char *base = static_cast<char *>(ws);
  if (k == 1) {
    const size_t vb = v_bytes(p, gfull), mb = m_bytes(p, gfull);
    return forward_one(p, gfull, x, U, y, base, reinterpret_cast<float *>(base + vb), s, s, s, nullptr, nullptr,
                       reinterpret_cast<int *>(base + vb + mb));
  }
  const int nc = (N + k - 1) / k;
  const int nchunks = (N + nc - 1) / nc;
  Geometry gc = make_geometry(p, nc, H, W);
  gc.gemm_ctas = env_int("NW_GEMM_CTAS", 0);
  const size_t vb = v_bytes(p, gc), mb = m_bytes(p, gc);
  const size_t es = (p->dtype == NW_DTYPE_BF16) ? 2 : 4;
  const size_t ximg = (size_t)p->Cin * H * W * es, yimg = (size_t)p->Cout * gfull.Ho * gfull.Wo * es;
  // streams and events of the pipeline (the plan's, created once; enqueued under pipe_mu,
  // which nw_conv_forward_host's io_mu nests around)
  std::lock_guard<std::mutex> lk(p->pipe_mu);
  for (auto &ps : p->s_pipe)
    if (!ps && cudaStreamCreateWithFlags(&ps, cudaStreamNonBlocking) != cudaSuccess) return NW_ERR_CUDA;
  cudaStream_t si = p->s_pipe[0], sg = p->s_pipe[1], so = p->s_pipe[2];
  // events: start, then per chunk in / gemm / out
  if (!ensure_events(p->ev_pipe, 1 + 3 * (size_t)nchunks)) return NW_ERR_CUDA;
  const std::vector<cudaEvent_t> &ev = p->ev_pipe;
  auto E_in = [&](int c) { return ev[1 + 3 * c]; };
  auto E_gemm = [&](int c) { return ev[2 + 3 * c]; };
  auto E_out = [&](int c) { return ev[3 + 3 * c]; };
  bool ok = cudaEventRecord(ev[0], s) == cudaSuccess;
  for (cudaStream_t t : {si, sg, so}) ok = ok && cudaStreamWaitEvent(t, ev[0], 0) == cudaSuccess;
  for (int c = 0; ok && st == NW_OK && c < nchunks; ++c) {
    const int n0 = c * nc, nk = (N - n0) < nc ? (N - n0) : nc, b = c & 1;
    Geometry g = (nk == nc) ? gc : make_geometry(p, nk, H, W);
    g.gemm_ctas = gc.gemm_ctas;
    char *V = base + (size_t)b * (vb + mb);
    float *M = reinterpret_cast<float *>(V + vb);
    if (c >= 2) {  // buffer b: V read by contraction c-2, M read by output transform c-2
      ok = ok && cudaStreamWaitEvent(si, E_gemm(c - 2), 0) == cudaSuccess;
      ok = ok && cudaStreamWaitEvent(sg, E_out(c - 2), 0) == cudaSuccess;
    }
    if (!ok) break;
    st = forward_one(p, g, static_cast<const char *>(x) + (size_t)n0 * ximg, U,
                     static_cast<char *>(y) + (size_t)n0 * yimg, V, M, si, sg, so, E_in(c), E_gemm(c));
    ok = ok && cudaEventRecord(E_out(c), so) == cudaSuccess;
  }
  if (ok && st == NW_OK) ok = cudaStreamWaitEvent(s, E_out(nchunks - 1), 0) == cudaSuccess;
  if (st != NW_OK) return st;
  return ok ? NW_OK : NW_ERR_CUDA;
}

}  // extern "C"

extern "C" {

// Host-buffer forward, pipelined: the batch is cut into chunks of nc images;
// chunk k's x is copied host -> device on a copy stream while chunk k-1 runs
// the nested forward on `stream` and chunk k-2's y is copied device -> host on
// a second copy stream (PCIe is full duplex).  x and y chunks are double
// buffered in the workspace; events order reuse.  The call stays asynchronous:
// `stream` waits for the last device -> host copy before anything enqueued
// after this call.
static int host_chunk(int N) {
  // images per full chunk: ~NW_HOST_CHUNKS chunks (default 8); the schedule ramps up and
  // down around it so the pipeline fill (first H2D) and drain (last D2H) stay short
  static const int k = env_int("NW_HOST_CHUNKS", 8);  // once per process: workspace sizes stay consistent
  int nc = (N + (k > 0 ? k : 1) - 1) / (k > 0 ? k : 1);
  return nc < 1 ? 1 : nc;
}

static void host_layout(const nw_plan_st *p, int N, int H, int W, size_t *fw, size_t *xb, size_t *yb, int *nc) {
  *nc = host_chunk(N);
  Geometry g = make_geometry(p, *nc, H, W);
  const size_t es = (p->dtype == NW_DTYPE_BF16) ? 2 : 4;
  *fw = forward_ws_bytes(p, *nc, H, W);
  *xb = (size_t)round_up((long long)*nc * p->Cin * H * W * es, 256);
  *yb = (size_t)round_up((long long)*nc * p->Cout * g.Ho * g.Wo * es, 256);
}

nw_plan_st::~nw_plan_st() {
  for (auto e : ev_host) cudaEventDestroy(e);
  for (auto e : ev_pipe) cudaEventDestroy(e);
  if (s_h2d) cudaStreamDestroy(s_h2d);
  if (s_d2h) cudaStreamDestroy(s_d2h);
  for (auto &ps : s_pipe)
    if (ps) cudaStreamDestroy(ps);
}

nw_status_t nw_workspace_size_host(nw_plan_t p, int N, int H, int W, size_t *bytes) {
  if (!p || !bytes || N < 1 || H < 1 || W < 1) return NW_ERR_INVALID;
  nw_status_t st = finalize(p);
  if (st != NW_OK) return st;
  Geometry g = make_geometry(p, N, H, W);
  if (g.Ho < 1 || g.Wo < 1) return NW_ERR_INVALID;
  size_t fw, xb, yb;
  int nc;
  host_layout(p, N, H, W, &fw, &xb, &yb, &nc);
  *bytes = fw + 2 * xb + 2 * yb;
  return NW_OK;
}

nw_status_t nw_conv_forward_host(nw_plan_t p, const void *x_host, const void *U, void *y_host, int N, int H, int W,
                                 void *ws, size_t ws_bytes, nw_stream_t stream) {
  if (!p || !x_host || !y_host || !U || N < 1 || H < 1 || W < 1) return NW_ERR_INVALID;
  size_t need = 0;
  nw_status_t st = nw_workspace_size_host(p, N, H, W, &need);
  if (st != NW_OK) return st;
  if (!ws || ws_bytes < need) return NW_ERR_WORKSPACE;
  size_t fw, xb, yb;
  int nc;
  host_layout(p, N, H, W, &fw, &xb, &yb, &nc);
  Geometry g = make_geometry(p, N, H, W);
  const size_t es = (p->dtype == NW_DTYPE_BF16) ? 2 : 4;
  const size_t ximg = (size_t)p->Cin * H * W * es, yimg = (size_t)p->Cout * g.Ho * g.Wo * es;
  char *base = static_cast<char *>(ws);
  char *xd[2] = {base + fw, base + fw + xb};
  char *yd[2] = {base + fw + 2 * xb, base + fw + 2 * xb + yb};
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  std::lock_guard<std::mutex> lk(p->io_mu);  // copy streams and the event pool (enqueue only)
  if (!p->s_h2d && cudaStreamCreateWithFlags(&p->s_h2d, cudaStreamNonBlocking) != cudaSuccess) return NW_ERR_CUDA;
  if (!p->s_d2h && cudaStreamCreateWithFlags(&p->s_d2h, cudaStreamNonBlocking) != cudaSuccess) return NW_ERR_CUDA;
  // chunk schedule: ramp 1, 2, 4 .. up to nc images, nc-image chunks, ramp back down, so the
  // unoverlapped first copy in and last copy out are one image each
  std::vector<int> sizes;
  {
    std::vector<int> head;
    int hs = 0;
    for (int c = 1; c < nc; c *= 2) { head.push_back(c); hs += c; }
    if (2 * hs >= N) {
      sizes.assign(N, 1);
    } else {
      sizes = head;
      int mid = N - 2 * hs;
      while (mid > 0) { const int c = mid < nc ? mid : nc; sizes.push_back(c); mid -= c; }
      sizes.insert(sizes.end(), head.rbegin(), head.rend());
    }
  }
  const int nchunks = (int)sizes.size();
  // events: [0] start, per chunk: in (x landed), comp (forward done), out (y copied); the
  // plan's pool, enqueued under io_mu
  if (!ensure_events(p->ev_host, 1 + 3 * (size_t)nchunks)) return NW_ERR_CUDA;
  const std::vector<cudaEvent_t> &ev = p->ev_host;
  auto E_in = [&](int k) { return ev[1 + 3 * k]; };
  auto E_comp = [&](int k) { return ev[2 + 3 * k]; };
  auto E_out = [&](int k) { return ev[3 + 3 * k]; };
  bool ok = cudaEventRecord(ev[0], s) == cudaSuccess && cudaStreamWaitEvent(p->s_h2d, ev[0], 0) == cudaSuccess &&
            cudaStreamWaitEvent(p->s_d2h, ev[0], 0) == cudaSuccess;
  int n0 = 0;
  for (int k = 0; ok && k < nchunks; n0 += sizes[k], ++k) {
    const int nk = sizes[k], b = k & 1;
    if (k >= 2) ok = ok && cudaStreamWaitEvent(p->s_h2d, E_comp(k - 2), 0) == cudaSuccess;  // x buffer free
    ok = ok && cudaMemcpyAsync(xd[b], static_cast<const char *>(x_host) + (size_t)n0 * ximg, (size_t)nk * ximg,
                               cudaMemcpyHostToDevice, p->s_h2d) == cudaSuccess;
    ok = ok && cudaEventRecord(E_in(k), p->s_h2d) == cudaSuccess;
    ok = ok && cudaStreamWaitEvent(s, E_in(k), 0) == cudaSuccess;
    if (k >= 2) ok = ok && cudaStreamWaitEvent(s, E_out(k - 2), 0) == cudaSuccess;  // y buffer free
    if (!ok) break;
    st = nw_conv_forward(p, xd[b], U, yd[b], nk, H, W, ws, fw, stream);
    if (st != NW_OK) break;
    ok = cudaEventRecord(E_comp(k), s) == cudaSuccess && cudaStreamWaitEvent(p->s_d2h, E_comp(k), 0) == cudaSuccess;
    ok = ok && cudaMemcpyAsync(static_cast<char *>(y_host) + (size_t)n0 * yimg, yd[b], (size_t)nk * yimg,
                               cudaMemcpyDeviceToHost, p->s_d2h) == cudaSuccess;
    ok = ok && cudaEventRecord(E_out(k), p->s_d2h) == cudaSuccess;
  }
  if (st == NW_OK && ok) ok = cudaStreamWaitEvent(s, E_out(nchunks - 1), 0) == cudaSuccess;
  if (st != NW_OK) return st;
  return ok ? NW_OK : NW_ERR_CUDA;
}

}  // extern "C"
