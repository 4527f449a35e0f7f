// comparison.cu -- the two comparison paths of the C ABI:
//   nw_conv_ola     OLA-Winograd (Eq. 2.3): the Kp-tap phase filter is cut
//                   into nb = ceil(Kp/3) blocks of 3 taps per axis, each run on a
//                   single-level F(3x3, 3x3) = F(1,1) (x) F(3,3) over the tile grid
//                   shifted by the block offset, and the nb^2 results are summed --
//                   in the contraction, whose K runs over (block, channel) with the
//                   A rows of block (bh, bw) read at tile t + bh * tiles_w + bw.
//   nw_conv_direct  native convolution (Eq. 2.1) as an implicit GEMM over the
//                   (phase) pixel grid: K runs over (tap, channel), tap (a, b) reads
//                   pixel row t + a * W_ext + b of a padded NHWC copy of x.
// Both reuse the nested path's kernels (filter transform with blocks, input /
// output transforms instantiated for F(1,1) (x) F(3,3), the tcgen05 or FP32
// contraction with shifted A rows) and run in the plan's math mode, so the
// three paths are compared at the same arithmetic.  The filter transform runs
// inside each call (into the workspace).
#include <cuda_bf16.h>

#include "ptx.cuh"
#include "transforms.cuh"

namespace nw {

// ---------------------------------------------------------------------------
// direct path: x NCHW -> V [T_pad][cin_pad] (bf16 hi / lo planes or fp32) on the
// extended phase-pixel grid; one block = 32 pixels of one grid row x all channels
// ---------------------------------------------------------------------------
template <typename XT, bool BF>
__global__ void __launch_bounds__(256) pack_input_kernel(const XT* __restrict__ x, void* __restrict__ Vout, Geometry g,
                                                         int wchunks) {
  extern __shared__ float sm[];  // [32][cin_pad + 1]
  const int cs = g.cin_pad + 1;
  int b = blockIdx.x;
  const int wc = b % wchunks;
  b /= wchunks;
  const int u = b % g.tiles_h;
  const int n = b / g.tiles_h;
  const int v0 = wc * 32;
  for (int i = threadIdx.x; i < 32 * g.cin_pad; i += blockDim.x) {
    const int j = i % 32, ce = i / 32;
    const int v = v0 + j;
    int ci = ce, p = 0, q = 0;
    if (g.mode == 1) {  // phase-major stride-2 channels: ce = (2p + q) * cs + ci
      const int phase = ce / g.cs;
      ci = phase < 4 ? ce - phase * g.cs : g.Cin;
      p = phase / 2;
      q = phase % 2;
    }
    const int r = g.SR * u + p + g.off[0], c = g.SR * v + q + g.off[0];
    float val = 0.f;
    if (v < g.tiles_w && ci < g.Cin && r >= 0 && r < g.H && c >= 0 && c < g.W)
      val = to_f(x[(((long long)n * g.Cin + ci) * g.H + r) * g.W + c]);
    sm[j * cs + ce] = val;
  }
  __syncthreads();
  const long long plane = (long long)g.T_pad * g.cin_pad;
  const int half = g.cin_pad / 2;
  for (int i = threadIdx.x; i < 32 * half; i += blockDim.x) {
    const int cp = i % half, j = i / half;
    const int v = v0 + j;
    if (v >= g.tiles_w) continue;
    const long long t = ((long long)n * g.tiles_h + u) * g.tiles_w + v;
    const float a = sm[j * cs + 2 * cp], bb = sm[j * cs + 2 * cp + 1];
    const long long o = t * g.cin_pad + 2 * cp;
    if (BF) {
      __nv_bfloat16* V = reinterpret_cast<__nv_bfloat16*>(Vout);
      uint32_t hi, lo;
      ptx::split_bf16x2(a, bb, hi, lo);
      *reinterpret_cast<uint32_t*>(V + o) = hi;
      *reinterpret_cast<uint32_t*>(V + plane + o) = lo;
    } else {
      *reinterpret_cast<float2*>(reinterpret_cast<float*>(Vout) + o) = make_float2(a, bb);
    }
  }
}

// M [cout_pad][T_pad] -> y NCHW (crop, transposed depth-to-space, PReLU, cast); one thread per y element
template <typename YT>
__global__ void __launch_bounds__(256) unpack_output_kernel(const float* __restrict__ M, YT* __restrict__ y, Geometry g,
                                                            const float* __restrict__ slopes) {
  const long long total = (long long)g.N * g.Cout * g.Ho * g.Wo;
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (long long)gridDim.x * blockDim.x) {
    const int X = (int)(e % g.Wo);
    long long r = e / g.Wo;
    const int Yr = (int)(r % g.Ho);
    r /= g.Ho;
    const int c = (int)(r % g.Cout);
    const int n = (int)(r / g.Cout);
    int i = Yr, j = X, coe = c;
    if (g.mode == 2) {
      i = Yr / 2;
      j = X / 2;
      coe = ((Yr % 2) * 2 + (X % 2)) * g.Cout + c;
    }
    const long long t = ((long long)n * g.tiles_h + i) * g.tiles_w + j;
    float v = M[(long long)coe * g.T_pad + t];
    if (slopes) v = v >= 0.f ? v : slopes[c] * v;
    y[e] = from_f<YT>(v);
  }
}

nw_status_t launch_pack_input(const nw_plan_st* p, const Geometry& g, const void* x, void* V, cudaStream_t s) {
  const int wchunks = (g.tiles_w + 31) / 32;
  const long long nb = (long long)g.N * g.tiles_h * wchunks;
  const size_t smem = (size_t)32 * (g.cin_pad + 1) * sizeof(float);
  if (nb >= (1ll << 31) || smem > 200 * 1024) return NW_ERR_UNSUPPORTED;
  const bool bf = p->math != NW_MATH_FP32_SIMT;
  LaunchScope scope_("pack_input", s);
  if (p->dtype == NW_DTYPE_BF16) {
    auto k = bf ? pack_input_kernel<__nv_bfloat16, true> : pack_input_kernel<__nv_bfloat16, false>;
    if ((bf ? ensure_smem<pack_input_kernel<__nv_bfloat16, true>>(200 * 1024)
            : ensure_smem<pack_input_kernel<__nv_bfloat16, false>>(200 * 1024)) != NW_OK)
      return NW_ERR_CUDA;
    k<<<(unsigned)nb, 256, smem, s>>>(static_cast<const __nv_bfloat16*>(x), V, g, wchunks);
  } else {
    auto k = bf ? pack_input_kernel<float, true> : pack_input_kernel<float, false>;
    if ((bf ? ensure_smem<pack_input_kernel<float, true>>(200 * 1024)
            : ensure_smem<pack_input_kernel<float, false>>(200 * 1024)) != NW_OK)
      return NW_ERR_CUDA;
    k<<<(unsigned)nb, 256, smem, s>>>(static_cast<const float*>(x), V, g, wchunks);
  }
  return check_launch();
}

nw_status_t launch_unpack_output(const nw_plan_st* p, const Geometry& g, const float* M, void* y, cudaStream_t s) {
  const long long total = (long long)g.N * g.Cout * g.Ho * g.Wo;
  long long blocks = (total + 255) / 256;
  if (blocks > 148 * 64) blocks = 148 * 64;
  const float* sl = p->prelu ? p->slopes : nullptr;
  LaunchScope scope_("unpack_output", s);
  if (p->dtype == NW_DTYPE_BF16)
    unpack_output_kernel<__nv_bfloat16><<<(unsigned)blocks, 256, 0, s>>>(M, static_cast<__nv_bfloat16*>(y), g, sl);
  else
    unpack_output_kernel<float><<<(unsigned)blocks, 256, 0, s>>>(M, static_cast<float*>(y), g, sl);
  return check_launch();
}

}  // namespace nw

using namespace nw;

namespace {

inline bool aligned16(const void* ptr) { return (reinterpret_cast<uintptr_t>(ptr) & 15u) == 0; }

nw_status_t comparison_ws(nw_plan_t p, int N, int H, int W, int path, size_t* bytes) {
  if (!p || !bytes || N < 1 || H < 1 || W < 1) return NW_ERR_INVALID;
  nw_status_t st = finalize(p);
  if (st != NW_OK) return st;
  Geometry g = make_geometry(p, N, H, W, path);
  if (g.Ho < 1 || g.Wo < 1) return NW_ERR_INVALID;
  if (g.nsh > kMaxShift) return NW_ERR_UNSUPPORTED;
  *bytes = u_bytes(g) + v_bytes(p, g) + m_bytes(p, g);
  return NW_OK;
}

nw_status_t run_comparison(nw_plan_t p, const void* x, const void* w, void* y, int N, int H, int W, void* ws,
                           size_t ws_bytes, nw_stream_t stream, int path) {
  if (!p || !x || !w || !y) return NW_ERR_INVALID;
  size_t need = 0;
  nw_status_t st = comparison_ws(p, N, H, W, path, &need);
  if (st != NW_OK) return st;
  if (!aligned16(x) || !aligned16(y) || !aligned16(ws)) return NW_ERR_INVALID;
  if (!ws || ws_bytes < need) return NW_ERR_WORKSPACE;
  Geometry g = make_geometry(p, N, H, W, path);
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  char* base = static_cast<char*>(ws);
  void* U = base;
  void* V = base + u_bytes(g);
  float* M = reinterpret_cast<float*>(base + u_bytes(g) + v_bytes(p, g));
  if ((st = launch_filter_transform(p, g, w, U, s)) != NW_OK) return st;
  st = (path == kPathDirect) ? launch_pack_input(p, g, x, V, s) : launch_input_transform(p, g, x, V, s);
  if (st != NW_OK) return st;
  if (p->depthwise)  // per-channel sum over the shifted blocks / taps (no channel contraction)
    st = launch_depthwise_product(p, g, V, static_cast<const float*>(U), M, s);
  else if (p->math == NW_MATH_FP32_SIMT)
    st = launch_gemm_simt(p, g, static_cast<const float*>(V), static_cast<const float*>(U), M, s);
  else
    st = launch_gemm_tc(p, g, V, U, M, s);
  if (st != NW_OK) return st;
  return (path == kPathDirect) ? launch_unpack_output(p, g, M, y, s) : launch_output_transform(p, g, M, y, s);
}

}  // namespace

extern "C" {

nw_status_t nw_workspace_size_ola(nw_plan_t p, int N, int H, int W, size_t* bytes) {
  return comparison_ws(p, N, H, W, kPathOla, bytes);
}
nw_status_t nw_workspace_size_direct(nw_plan_t p, int N, int H, int W, size_t* bytes) {
  return comparison_ws(p, N, H, W, kPathDirect, bytes);
}
nw_status_t nw_conv_ola(nw_plan_t p, const void* x, const void* w, void* y, int N, int H, int W, void* ws,
                        size_t ws_bytes, nw_stream_t stream) {
  return run_comparison(p, x, w, y, N, H, W, ws, ws_bytes, stream, kPathOla);
}
nw_status_t nw_conv_direct(nw_plan_t p, const void* x, const void* w, void* y, int N, int H, int W, void* ws,
                           size_t ws_bytes, nw_stream_t stream) {
  return run_comparison(p, x, w, y, N, H, W, ws, ws_bytes, stream, kPathDirect);
}

}  // extern "C"
