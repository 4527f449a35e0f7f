// transforms.cuh -- shared device helpers of the SIMT kernels of the nested-Winograd pipeline (sm_100a):
//   G1 filter transform   U = G_hat W G_hat^T
//   G2 input transform    V = B^T_hat X B_hat per slice
//   G3s FP32 contraction  M_xi = V_xi . U_xi^T for every point  (Eq. 2.1 channel sum)
//   G4 output transform   Y = A^T_hat M A_hat + scatter/keep + store
// The transforms are compile-time (constexpr Cook-Toom, cooktoom.cuh), applied
// per axis in the factored two-level form (B_o^T (x) B_i^T: inner F(m_i,3) on each
// reordered column, then outer F(m_o,r_o) across columns) so zero entries and
// +-1 coefficients vanish from the instruction stream.
#pragma once
#include <cuda_bf16.h>

#include "nw_internal.h"

namespace nw {

template <int MO, int RO, int MI>
struct Ax {
  static constexpr NestedAxis A = make_axis(MO, RO, MI);
  static constexpr int LO = A.l_o, LI = A.l_i, PA = A.Pa, L = A.L, MA = A.Ma, R = A.R;
  static constexpr int ADV = A.adv, NPH = A.nph, SHMAX = A.shift[A.nph - 1];
};

// ---------------------------------------------------------------------------
// per-axis transforms (factored), float
// ---------------------------------------------------------------------------
// x[L] (slice window along one axis) -> v[PA] = B^T_hat x
template <int MO, int RO, int MI>
__device__ __forceinline__ void in_axis(const float* x, float* v) {
  using X = Ax<MO, RO, MI>;
  constexpr AxisF F = axis_f(MO, RO, MI);
  float z[X::LO][X::LI];
#pragma unroll
  for (int j = 0; j < X::LO; ++j)
#pragma unroll
    for (int pi = 0; pi < X::LI; ++pi) {
      float acc = 0.f;
      bool first = true;
#pragma unroll
      for (int s = 0; s < X::LI; ++s) {
        if (F.BiT[pi][s] != 0.f) {
          const float t = F.BiT[pi][s] * x[kRi * j + s];
          acc = first ? t : acc + t;
          first = false;
        }
      }
      z[j][pi] = acc;
    }
#pragma unroll
  for (int po = 0; po < X::LO; ++po)
#pragma unroll
    for (int pi = 0; pi < X::LI; ++pi) {
      float acc = 0.f;
      bool first = true;
#pragma unroll
      for (int j = 0; j < X::LO; ++j) {
        if (F.BoT[po][j] != 0.f) {
          const float t = F.BoT[po][j] * z[j][pi];
          acc = first ? t : acc + t;
          first = false;
        }
      }
      v[po * X::LI + pi] = acc;
    }
}

// m[PA] -> y[MA] = A^T_hat m
template <int MO, int RO, int MI>
__device__ __forceinline__ void out_axis(const float* m, float* y) {
  using X = Ax<MO, RO, MI>;
  constexpr AxisF F = axis_f(MO, RO, MI);
  float u[X::LO][MI];
#pragma unroll
  for (int po = 0; po < X::LO; ++po)
#pragma unroll
    for (int s = 0; s < MI; ++s) {
      float acc = 0.f;
      bool first = true;
#pragma unroll
      for (int pi = 0; pi < X::LI; ++pi) {
        if (F.AiT[s][pi] != 0.f) {
          const float t = F.AiT[s][pi] * m[po * X::LI + pi];
          acc = first ? t : acc + t;
          first = false;
        }
      }
      u[po][s] = acc;
    }
#pragma unroll
  for (int t = 0; t < MO; ++t)
#pragma unroll
    for (int s = 0; s < MI; ++s) {
      float acc = 0.f;
      bool first = true;
#pragma unroll
      for (int po = 0; po < X::LO; ++po) {
        if (F.AoT[t][po] != 0.f) {
          const float v = F.AoT[t][po] * u[po][s];
          acc = first ? v : acc + v;
          first = false;
        }
      }
      y[t * MI + s] = acc;
    }
}

template <typename T>
__device__ __forceinline__ float to_f(T v);
template <>
__device__ __forceinline__ float to_f<float>(float v) { return v; }
template <>
__device__ __forceinline__ float to_f<__nv_bfloat16>(__nv_bfloat16 v) { return __bfloat162float(v); }

template <typename T>
__device__ __forceinline__ T from_f(float v);
template <>
__device__ __forceinline__ float from_f<float>(float v) { return v; }
template <>
__device__ __forceinline__ __nv_bfloat16 from_f<__nv_bfloat16>(float v) { return __float2bfloat16_rn(v); }

}  // namespace nw
