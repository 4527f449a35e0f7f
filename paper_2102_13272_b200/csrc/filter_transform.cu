// filter_transform.cu -- G1: nested filter transform.
// Per (output channel, input channel) pair of the phase-folded layer: gather the
// phase sub-filter (Eq. 2.7 taps, or the flipped taps of a transposed phase),
// zero-pad it "at the end" to 3r_o x 3r_o, and compute
// U = G_hat W G_hat^T in fp64, rounded once to fp32 or to a bf16 hi/lo pair.
// G_hat (P_a x 3r_o, fp64) comes from the planner through the kernel parameters.
#include <cuda_bf16.h>

#include "nw_internal.h"

namespace nw {

struct GhatParam {
  double g[kMaxPa * kMaxR];
  int Pa, R;
};

template <typename WT>
__device__ __forceinline__ double ld_w(const WT* w, long long i);
template <>
__device__ __forceinline__ double ld_w<float>(const float* w, long long i) { return (double)w[i]; }
template <>
__device__ __forceinline__ double ld_w<__nv_bfloat16>(const __nv_bfloat16* w, long long i) {
  return (double)__bfloat162float(w[i]);
}

template <typename WT, bool BF>
__global__ void __launch_bounds__(128) filter_transform_kernel(const WT* __restrict__ w, void* __restrict__ Uout,
                                                               Geometry g, int K, const __grid_constant__ GhatParam G) {
  // one thread per (output channel coe, filter block b, contraction channel ce);
  // U layout [P][cout_pad][nsh * cin_pad], K index = b * cin_pad + ce
  const long long kdim = (long long)g.nsh * g.cin_pad;
  const long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (long long)g.cout_pad * kdim) return;
  const int kk = (int)(idx % kdim);
  const int coe = (int)(idx / kdim);
  const int ce = kk % g.cin_pad, blk = kk / g.cin_pad;
  const int bh = blk / g.nb, bw = blk % g.nb;
  const int R = G.R, Pa = G.Pa;
  double We[kMaxR * kMaxR];
  for (int i = 0; i < R * R; ++i) We[i] = 0.0;
  int ci = ce, ph = 0, pw = 0;
  if (g.mode == 1) {  // phase-major stride-2 channels: ce = (2 ph + pw) * cs + ci
    const int phase = ce / g.cs;
    ci = ce - phase * g.cs;
    ph = phase / 2;
    pw = phase % 2;
    if (phase >= 4) ci = g.Cin;  // padding channel
  }
  if (ci < g.Cin && ce < g.cin_pad && coe < g.cout_e) {
    int co = coe;
    if (g.mode == 2) { const int f = coe / g.Cout; co = coe % g.Cout; ph = f / 2; pw = f % 2; }
    for (int a = 0; a < R; ++a)
      for (int b = 0; b < R; ++b) {
        const int ka = bh * R + a, kb = bw * R + b;   // phase-filter taps of this block (zero past Kp: P:106)
        if (ka >= g.Kp || kb >= g.Kp) continue;
        const int th = g.taps[ph][ka], tw = g.taps[pw][kb];
        if (th < 0 || tw < 0) continue;
        const long long off = (g.mode == 2) ? (((long long)ci * g.Cout + co) * K + th) * K + tw
                                            : (((long long)co * g.Cin + ci) * K + th) * K + tw;
        We[a * R + b] = ld_w(w, off);
      }
  }
  const long long rowlen = (long long)g.cout_pad * kdim;       // elements per point
  const long long plane = (long long)Pa * Pa * rowlen;
  double t1[kMaxR];
  for (int p1 = 0; p1 < Pa; ++p1) {
    for (int b = 0; b < R; ++b) {
      double acc = 0.0;
      for (int a = 0; a < R; ++a) acc += G.g[p1 * R + a] * We[a * R + b];
      t1[b] = acc;
    }
    for (int p2 = 0; p2 < Pa; ++p2) {
      double u = 0.0;
      for (int b = 0; b < R; ++b) u += t1[b] * G.g[p2 * R + b];
      const long long o = (long long)(p1 * Pa + p2) * rowlen + (long long)coe * kdim + kk;
      if (BF) {
        __nv_bfloat16* U = reinterpret_cast<__nv_bfloat16*>(Uout);
        const __nv_bfloat16 hi = __double2bfloat16(u);
        const __nv_bfloat16 lo = __double2bfloat16(u - (double)__bfloat162float(hi));
        U[o] = hi;
        U[plane + o] = lo;
      } else {
        reinterpret_cast<float*>(Uout)[o] = (float)u;
      }
    }
  }
}

nw_status_t launch_filter_transform(const nw_plan_st* p, const Geometry& g_in, const void* w, void* U,
                                    cudaStream_t s) {
  Geometry g = g_in;
  if (p->depthwise) {  // w [C][1][K][K]: one single-input-channel filter per channel -> U [P][cout_pad][nsh]
    g.Cin = 1;
    g.cin_e = 1;
    g.cin_pad = 1;
  }
  GhatParam G{};
  const NestedAxis ax = path_axis(p, g.path);
  G.Pa = ax.Pa;
  G.R = g.R;
  for (int q = 0; q < G.Pa; ++q)
    for (int k = 0; k < G.R; ++k) G.g[q * G.R + k] = (g.path == kPathDirect) ? 1.0 : rdouble(g_hat(ax, q, k));
  const long long n = (long long)g.cout_pad * g.nsh * g.cin_pad;
  const int blocks = (int)((n + 127) / 128);
  const bool bf = p->math != NW_MATH_FP32_SIMT && !p->depthwise;  // depthwise U stays fp32
  LaunchScope scope_("filter_transform", s);
  if (p->dtype == NW_DTYPE_BF16) {
    const __nv_bfloat16* wb = static_cast<const __nv_bfloat16*>(w);
    if (bf) filter_transform_kernel<__nv_bfloat16, true><<<blocks, 128, 0, s>>>(wb, U, g, p->K, G);
    else filter_transform_kernel<__nv_bfloat16, false><<<blocks, 128, 0, s>>>(wb, U, g, p->K, G);
  } else {
    const float* wf = static_cast<const float*>(w);
    if (bf) filter_transform_kernel<float, true><<<blocks, 128, 0, s>>>(wf, U, g, p->K, G);
    else filter_transform_kernel<float, false><<<blocks, 128, 0, s>>>(wf, U, g, p->K, G);
  }
  return check_launch();
}

}  // namespace nw
