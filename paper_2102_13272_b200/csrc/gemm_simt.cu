// gemm_simt.cu -- G3s FP32 CUDA-core contraction (the accuracy reference path)
#include "nw_internal.h"

namespace nw {

// ---------------------------------------------------------------------------
// G3s: FP32 SIMT contraction, batched over transform points
// M[xi][co][t] = sum_k V[xi][t][k] * U[xi][co][k]
// The channel sum is accumulated in FP64: the product of two fp32 operands is exact in fp64,
// so M carries one rounding (to fp32, at the store) instead of one per channel.  With fp32
// accumulation the FP32 path measured 1.12e-4 on C3 at full size (Cin = 256, nested
// F(4,3) (x) F(3,3): the output transform amplifies the M rounding), above the 1e-4 gate;
// a CPU split of the error (fp32 V / U / M separately) put 90 % of it in the accumulation.
// ---------------------------------------------------------------------------
struct Shifts {
  int nsh, cin_pad;
  int off[kMaxShift];
};

// K = nsh * cin_pad: k-range of shift s reads A rows t + off[s] (OLA / direct
// comparison paths); rows past the point's T_pad read as zero.
__global__ void __launch_bounds__(256) gemm_simt_kernel(const float* __restrict__ V, const float* __restrict__ U,
                                                        float* __restrict__ M, long long T_pad, int K, int Nn,
                                                        const __grid_constant__ Shifts sh) {
  __shared__ float As[16][64 + 4];
  __shared__ float Bs[16][64 + 4];
  const int xi = blockIdx.z;
  const long long t0 = (long long)blockIdx.x * 64;
  const int n0 = blockIdx.y * 64;
  const int tid = threadIdx.x, ty = tid / 16, tx = tid % 16;
  const float* Vb = V + (long long)xi * T_pad * sh.cin_pad;
  const float* Ub = U + ((long long)xi * Nn + n0) * K;
  double acc[4][4] = {};
  const int lr = tid / 4, lk = (tid % 4) * 4;
  for (int k0 = 0; k0 < K; k0 += 16) {
    const int s = k0 / sh.cin_pad, kc = k0 - s * sh.cin_pad;
    const long long row = t0 + lr + sh.off[s];
    float4 a = make_float4(0.f, 0.f, 0.f, 0.f);
    if (row < T_pad) a = *reinterpret_cast<const float4*>(Vb + row * sh.cin_pad + kc + lk);
    float4 bb = make_float4(0.f, 0.f, 0.f, 0.f);
    if (n0 + lr < Nn) bb = *reinterpret_cast<const float4*>(Ub + (long long)lr * K + k0 + lk);
    As[lk + 0][lr] = a.x; As[lk + 1][lr] = a.y; As[lk + 2][lr] = a.z; As[lk + 3][lr] = a.w;
    Bs[lk + 0][lr] = bb.x; Bs[lk + 1][lr] = bb.y; Bs[lk + 2][lr] = bb.z; Bs[lk + 3][lr] = bb.w;
    __syncthreads();
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      float ar[4], br[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) ar[i] = As[k][ty * 4 + i];
#pragma unroll
      for (int j = 0; j < 4; ++j) br[j] = Bs[k][tx * 4 + j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fma((double)ar[i], (double)br[j], acc[i][j]);
    }
    __syncthreads();
  }
  // M layout [xi][co][t]: four consecutive slices per float4
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const int co = n0 + tx * 4 + j;
    if (co < Nn) {
      float* dst = M + ((long long)xi * Nn + co) * T_pad + t0 + ty * 4;
      *reinterpret_cast<float4*>(dst) =
          make_float4((float)acc[0][j], (float)acc[1][j], (float)acc[2][j], (float)acc[3][j]);
    }
  }
}

nw_status_t launch_gemm_simt(const nw_plan_st* p, const Geometry& g, const float* V, const float* U, float* M,
                             cudaStream_t s) {
  (void)p;
  dim3 grid((unsigned)(g.T_pad / 64), (unsigned)((g.cout_pad + 63) / 64), (unsigned)g.P);
  LaunchScope scope_("contraction_fp32_simt", s);
  Shifts sh{};
  if (g.nsh < 1 || g.nsh > kMaxShift) return NW_ERR_UNSUPPORTED;
  sh.nsh = g.nsh;
  sh.cin_pad = g.cin_pad;
  for (int b = 0; b < g.nsh; ++b) sh.off[b] = (b / g.nb) * g.tiles_w + (b % g.nb);
  gemm_simt_kernel<<<grid, 256, 0, s>>>(V, U, M, g.T_pad, g.nsh * g.cin_pad, g.cout_pad, sh);
  return check_launch();
}

}  // namespace nw
