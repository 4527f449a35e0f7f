// depthwise.cu -- the per-channel transform-domain product of a depthwise layer (Table I's
// PNASNet depthwise 7x7 row).
//
// A depthwise convolution has no channel contraction (channel c of y sees only channel c of x
// and filter c), so Eq. 2.1's channel sum -- the GEMM of the nested path -- degenerates to the
// EWMM of P:110 alone:  M_xi[c][t] = V_xi[t][c] * U_xi[c].  The nested input and output
// transforms are the regular kernels (Cin = Cout = C); this kernel sits between them.  The
// OLA (Eq. 2.3) and direct (Eq. 2.1) comparison paths keep their sum over filter blocks /
// taps, which for a depthwise layer is a per-channel sum over shifted rows:
//     M_xi[c][t] = sum_b V_xi[t + off_b][c] * U_xi[c][b].
// One CTA per (128-slice block, point): products accumulate in a shared [128][C] tile, which
// is written transposed into M's [P][cout_pad][T_pad] rows with 16-byte stores.  HBM-bound
// (V read once per shift -- L2 hits after the first --, M written once).  Arithmetic: fp32
// products of v (fp32, hi + lo of the bf16x3 split -- exact in fp32 --, or hi alone for plain
// bf16) and the fp32 U of the depthwise filter transform.
#include <cuda_bf16.h>

#include "nw_internal.h"

namespace nw {

constexpr int kDwThreads = 256;

struct DwShifts {
  int nsh;
  int off[kMaxShift];
};

// VMODE 0: fp32 V [P][T_pad][cin_pad];  1: bf16 hi / lo planes [2][P][T_pad][cin_pad];
//       2: bf16 hi plane only;  3: blocked bf16x3 [T_pad/128][P][2][128][cin_pad] (nested)
// U: fp32 [P][cout_pad][nsh];  M: fp32 [P][cout_pad][T_pad]
template <int VMODE>
__global__ void __launch_bounds__(kDwThreads) depthwise_product_kernel(const void* __restrict__ V,
                                                                         const float* __restrict__ U,
                                                                         float* __restrict__ M, Geometry g,
                                                                         const __grid_constant__ DwShifts sh) {
  extern __shared__ float tile[];  // [128][cin_pad + 1]
  const int cpad = g.cin_pad, tstr = cpad + 1;
  const long long blk = blockIdx.x, xi = blockIdx.y;
  const int tid = threadIdx.x;
  const float* Ux = U + xi * g.cout_pad * sh.nsh;
  const int per_row = cpad / 8;
  for (int i = tid; i < 128 * per_row; i += kDwThreads) {
    const int r = i / per_row, c0 = (i % per_row) * 8;
    float acc[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) acc[k] = 0.f;
    for (int b = 0; b < sh.nsh; ++b) {
      const long long t = blk * 128 + r + sh.off[b];
      if (t >= g.T_pad) continue;  // rows past the point's slices read as zero
      float v[8];
      if constexpr (VMODE == 0) {
        const float* base = static_cast<const float*>(V) + (xi * g.T_pad + t) * (long long)cpad + c0;
        const float4 a = *reinterpret_cast<const float4*>(base), c = *reinterpret_cast<const float4*>(base + 4);
        v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w; v[4] = c.x; v[5] = c.y; v[6] = c.z; v[7] = c.w;
      } else {
        const __nv_bfloat16* base;
        long long lo_off;
        if constexpr (VMODE == 3) {
          base = static_cast<const __nv_bfloat16*>(V) + (((blk * g.P + xi) * 2) * 128 + r) * (long long)cpad + c0;
          lo_off = 128ll * cpad;
        } else {
          base = static_cast<const __nv_bfloat16*>(V) + (xi * g.T_pad + t) * (long long)cpad + c0;
          lo_off = (long long)g.P * g.T_pad * cpad;
        }
        const uint4 hi = *reinterpret_cast<const uint4*>(base);
        const __nv_bfloat16* h = reinterpret_cast<const __nv_bfloat16*>(&hi);
#pragma unroll
        for (int k = 0; k < 8; ++k) v[k] = __bfloat162float(h[k]);
        if constexpr (VMODE != 2) {
          const uint4 lo = *reinterpret_cast<const uint4*>(base + lo_off);
          const __nv_bfloat16* l = reinterpret_cast<const __nv_bfloat16*>(&lo);
#pragma unroll
          for (int k = 0; k < 8; ++k) v[k] += __bfloat162float(l[k]);
        }
      }
#pragma unroll
      for (int k = 0; k < 8; ++k) acc[k] = fmaf(v[k], Ux[(c0 + k) * sh.nsh + b], acc[k]);
    }
#pragma unroll
    for (int k = 0; k < 8; ++k) tile[r * tstr + c0 + k] = acc[k];
  }
  __syncthreads();
  // M row (xi, c) over the block's 128 slices, 4 slices per 16-byte store
  for (int i = tid; i < g.cout_e * 32; i += kDwThreads) {
    const int c = i / 32, r4 = (i % 32) * 4;
    const float4 o = make_float4(tile[(r4 + 0) * tstr + c], tile[(r4 + 1) * tstr + c], tile[(r4 + 2) * tstr + c],
                                 tile[(r4 + 3) * tstr + c]);
    *reinterpret_cast<float4*>(M + (xi * g.cout_pad + c) * g.T_pad + blk * 128 + r4) = o;
  }
}

nw_status_t launch_depthwise_product(const nw_plan_st* p, const Geometry& g, const void* V, const float* U, float* M,
                                     cudaStream_t s) {
  if (g.cin_pad % 8 != 0 || g.T_pad % 128 != 0 || g.nsh < 1 || g.nsh > kMaxShift) return NW_ERR_UNSUPPORTED;
  const size_t smem = (size_t)128 * (g.cin_pad + 1) * sizeof(float);
  if (smem > 227 * 1024) return NW_ERR_UNSUPPORTED;
  DwShifts sh{};
  sh.nsh = g.nsh;
  for (int b = 0; b < g.nsh; ++b) sh.off[b] = (b / g.nb) * g.tiles_w + (b % g.nb);
  const dim3 grid((unsigned)(g.T_pad / 128), (unsigned)g.P);
  // the opt-in limit is set once per device (ensure_smem): set it to the maximum, not this call's size
  constexpr int kMaxSmem = 227 * 1024;
  LaunchScope scope_("depthwise_product", s);
  const int vmode = g.vblk ? 3 : (p->math == NW_MATH_FP32_SIMT ? 0 : (p->math == NW_MATH_BF16 ? 2 : 1));
  switch (vmode) {
    case 0:
      if (ensure_smem<depthwise_product_kernel<0>>(kMaxSmem) != NW_OK) return NW_ERR_CUDA;
      depthwise_product_kernel<0><<<grid, kDwThreads, smem, s>>>(V, U, M, g, sh);
      break;
    case 1:
      if (ensure_smem<depthwise_product_kernel<1>>(kMaxSmem) != NW_OK) return NW_ERR_CUDA;
      depthwise_product_kernel<1><<<grid, kDwThreads, smem, s>>>(V, U, M, g, sh);
      break;
    case 2:
      if (ensure_smem<depthwise_product_kernel<2>>(kMaxSmem) != NW_OK) return NW_ERR_CUDA;
      depthwise_product_kernel<2><<<grid, kDwThreads, smem, s>>>(V, U, M, g, sh);
      break;
    default:
      if (ensure_smem<depthwise_product_kernel<3>>(kMaxSmem) != NW_OK) return NW_ERR_CUDA;
      depthwise_product_kernel<3><<<grid, kDwThreads, smem, s>>>(V, U, M, g, sh);
      break;
  }
  return check_launch();
}

}  // namespace nw
