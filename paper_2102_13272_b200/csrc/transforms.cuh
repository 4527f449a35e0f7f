// transforms.cuh -- shared device helpers of the SIMT kernels of the nested-Winograd pipeline (sm_100a):
//   G1 filter transform   U = G_hat W G_hat^T
//   G2 input transform    V = B^T_hat X B_hat per slice
//   G3s FP32 contraction  M_xi = V_xi . U_xi^T for every point  (Eq. 2.1 channel sum)
//   G4 output transform   Y = A^T_hat M A_hat + scatter/keep + store
// The transforms are compile-time (constexpr Cook-Toom, cooktoom.cuh), applied
// per axis in the factored two-level form (B_o^T (x) B_i^T: inner F(m_i,3) on each
// reordered column, then outer F(m_o,r_o) across columns).  Each level is one
// 1-D kernel (K1<m,r>::bt / ::at): generic kernels skip zero and +-1 coefficients at
// compile time; F(3,3) -- the kernel at both levels of the default plan -- and
// F(4,3) have hand-factored forms with shared subexpressions (F(3,3): 9 instead
// of 18 operations for B^T, 7 instead of 11 for A^T; F(4,3): 12 and 10).  Float addition is not associative, so the
// compiler cannot find these factorizations itself; the rounding order differs
// from the plain matrix product by a few ulp, far inside the accuracy budget.
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
// f2: two fp32 lanes in one 64-bit register, operated on by Blackwell's packed fp32
// instructions (add / sub / fma .rn.f32x2 -> SASS FADD2 / FFMA2).  Each lane is rounded exactly
// like the scalar instruction, so a packed transform of two independent columns gives the same
// bits as two scalar ones while issuing half the instructions (measured: FFMA2 sustains the
// same fp32 rate as FFMA, tools/ffma2_bench.cu).  Only add, sub and fma are provided (no
// separate multiply that ptxas could contract differently from the scalar code).
// ---------------------------------------------------------------------------
struct f2 {
  unsigned long long v;
};
__device__ __forceinline__ f2 f2_pack(float lo, float hi) {
  f2 r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r.v) : "f"(lo), "f"(hi));
  return r;
}
__device__ __forceinline__ void f2_unpack(f2 x, float& lo, float& hi) {
  asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(x.v));
}
__device__ __forceinline__ f2 f2_splat(float c) { return f2_pack(c, c); }
// the scalar fmaf stays visible next to the packed overload inside namespace nw
__device__ __forceinline__ float fmaf(float c, float x, float y) { return ::fmaf(c, x, y); }
__device__ __forceinline__ f2 operator+(f2 a, f2 b) {
  f2 r;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r.v) : "l"(a.v), "l"(b.v));
  return r;
}
__device__ __forceinline__ f2 operator-(f2 a, f2 b) {
  f2 r;
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r.v) : "l"(a.v), "l"(b.v));
  return r;
}
// -a as (-0) - a: exact, including the sign of zero
__device__ __forceinline__ f2 operator-(f2 a) { return f2_splat(-0.f) - a; }
__device__ __forceinline__ f2 fmaf(float c, f2 x, f2 y) {
  f2 r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r.v) : "l"(f2_splat(c).v), "l"(x.v), "l"(y.v));
  return r;
}

// ---------------------------------------------------------------------------
// one-level 1-D kernels: out[l] = B^T in[l] (l = m + r - 1), out[m] = A^T in[l]
// ---------------------------------------------------------------------------
template <int M, int R>
struct K1 {
  static constexpr int L = M + R - 1;
  static constexpr bool kPackedBt = false;  // scalar only (generic coefficient loop)
  __device__ __forceinline__ static void bt(const float (&x)[L], float (&o)[L]) {
    constexpr Kernel1D K = make_kernel(M, R);
#pragma unroll
    for (int i = 0; i < L; ++i) {
      float acc = 0.f;
      bool first = true;
#pragma unroll
      for (int j = 0; j < L; ++j) {
        const float c = float(rdouble(K.BT[i][j]));
        if (c != 0.f) {
          const float t = (c == 1.f) ? x[j] : (c == -1.f) ? -x[j] : c * x[j];
          acc = first ? t : ((c == -1.f) ? acc - x[j] : (c == 1.f) ? acc + x[j] : fmaf(c, x[j], acc));
          first = false;
        }
      }
      o[i] = acc;
    }
  }
  __device__ __forceinline__ static void at(const float (&x)[L], float (&o)[M]) {
    constexpr Kernel1D K = make_kernel(M, R);
#pragma unroll
    for (int i = 0; i < M; ++i) {
      float acc = 0.f;
      bool first = true;
#pragma unroll
      for (int j = 0; j < L; ++j) {
        const float c = float(rdouble(K.AT[i][j]));
        if (c != 0.f) {
          const float t = (c == 1.f) ? x[j] : (c == -1.f) ? -x[j] : c * x[j];
          acc = first ? t : ((c == -1.f) ? acc - x[j] : (c == 1.f) ? acc + x[j] : fmaf(c, x[j], acc));
          first = false;
        }
      }
      o[i] = acc;
    }
  }
};

// F(3,3), points {0, 1, -1, 2, inf} (R2):
//   B^T = [2 -1 -2 1 0; 0 2 1 -1 0; 0 -2 3 -1 0; 0 -1 0 1 0; 0 2 -1 -2 1]
//   A^T = [1 1 1 1 0; 0 1 -1 2 0; 0 1 1 4 1]
template <>
struct K1<3, 3> {
  static constexpr int L = 5;
  static constexpr bool kPackedBt = true;  // bt accepts f2 (packed pairs of columns)
  template <typename T>
  __device__ __forceinline__ static void bt(const T (&x)[5], T (&o)[5]) {
    const T a = x[3] - x[1];                             // row 3
    o[3] = a;
    o[0] = fmaf(2.f, x[0] - x[2], a);                    // 2x0 - x1 - 2x2 + x3
    o[1] = (x[1] + x[2]) - a;                            // 2x1 + x2 - x3
    o[2] = fmaf(2.f, fmaf(-2.f, x[1], x[2]), o[1]);      // -2x1 + 3x2 - x3
    o[4] = fmaf(-2.f, a, x[4] - x[2]);                   // 2x1 - x2 - 2x3 + x4
  }
  __device__ __forceinline__ static void at(const float (&x)[5], float (&o)[3]) {
    const float s = x[1] + x[2], d = x[1] - x[2];
    o[0] = (x[0] + x[3]) + s;                            // x0 + x1 + x2 + x3
    o[1] = fmaf(2.f, x[3], d);                           // x1 - x2 + 2x3
    o[2] = fmaf(4.f, x[3], s) + x[4];                    // x1 + x2 + 4x3 + x4
  }
};

// F(4,3), points {0, 1, -1, 2, -2, inf}:
//   B^T = [4 0 -5 0 1 0; 0 4 4 -1 -1 0; 0 -4 4 1 -1 0; 0 -2 -1 2 1 0; 0 2 -1 -2 1 0; 0 4 0 -5 0 1]
//   A^T = [1 1 1 1 1 0; 0 1 -1 2 -2 0; 0 1 1 4 4 0; 0 1 -1 8 -8 1]
template <>
struct K1<4, 3> {
  static constexpr int L = 6;
  static constexpr bool kPackedBt = true;
  template <typename T>
  __device__ __forceinline__ static void bt(const T (&x)[6], T (&o)[6]) {
    const T a = fmaf(-4.f, x[2], x[4]);                  // x4 - 4x2
    const T b = fmaf(-4.f, x[1], x[3]);                  // x3 - 4x1
    const T c = x[4] - x[2], d = x[3] - x[1];
    o[0] = fmaf(4.f, x[0], fmaf(-5.f, x[2], x[4]));      // 4x0 - 5x2 + x4
    o[1] = -a - b;                                       // 4x1 + 4x2 - x3 - x4
    o[2] = b - a;                                        // -4x1 + 4x2 + x3 - x4
    o[3] = fmaf(2.f, d, c);                              // -2x1 - x2 + 2x3 + x4
    o[4] = fmaf(-2.f, d, c);                             // 2x1 - x2 - 2x3 + x4
    o[5] = fmaf(4.f, x[1], fmaf(-5.f, x[3], x[5]));      // 4x1 - 5x3 + x5
  }
  __device__ __forceinline__ static void at(const float (&x)[6], float (&o)[4]) {
    const float s1 = x[1] + x[2], d1 = x[1] - x[2], s2 = x[3] + x[4], d2 = x[3] - x[4];
    o[0] = (x[0] + s1) + s2;                             // x0 + x1 + x2 + x3 + x4
    o[1] = fmaf(2.f, d2, d1);                            // x1 - x2 + 2x3 - 2x4
    o[2] = fmaf(4.f, s2, s1);                            // x1 + x2 + 4x3 + 4x4
    o[3] = fmaf(8.f, d2, d1) + x[5];                     // x1 - x2 + 8x3 - 8x4 + x5
  }
};

// Factored kernels are checked at compile time against the exact Cook-Toom tables (plan.cu's
// source of truth): the table a specialization hard-codes must equal make_kernel's.
__host__ __device__ constexpr bool bt_equal(int m1, int r1, int m2, int r2) {
  const Kernel1D a = make_kernel(m1, r1), b = make_kernel(m2, r2);
  if (a.l != b.l) return false;
  for (int i = 0; i < a.l; ++i)
    for (int j = 0; j < a.l; ++j)
      if (rdouble(a.BT[i][j]) != rdouble(b.BT[i][j])) return false;
  return true;
}
template <int M, int L>
__host__ __device__ constexpr bool at_equals(int r, const int (&t)[M][L]) {
  const Kernel1D k = make_kernel(M, r);
  if (k.l != L) return false;
  for (int i = 0; i < M; ++i)
    for (int j = 0; j < L; ++j)
      if (rdouble(k.AT[i][j]) != double(t[i][j])) return false;
  return true;
}

// F(4,2): points {0, 1, -1, 2, inf}, the point set of F(3,3), so B^T is F(3,3)'s
//   A^T = [1 1 1 1 0; 0 1 -1 2 0; 0 1 1 4 0; 0 1 -1 8 1]
constexpr int kAT42[4][5] = {{1, 1, 1, 1, 0}, {0, 1, -1, 2, 0}, {0, 1, 1, 4, 0}, {0, 1, -1, 8, 1}};
static_assert(bt_equal(4, 2, 3, 3) && at_equals<4, 5>(2, kAT42), "F(4,2) tables");
template <>
struct K1<4, 2> {
  static constexpr int L = 5;
  static constexpr bool kPackedBt = true;
  template <typename T>
  __device__ __forceinline__ static void bt(const T (&x)[5], T (&o)[5]) { K1<3, 3>::bt(x, o); }
  __device__ __forceinline__ static void at(const float (&x)[5], float (&o)[4]) {
    const float s = x[1] + x[2], d = x[1] - x[2];
    o[0] = (x[0] + x[3]) + s;                            // x0 + x1 + x2 + x3
    o[1] = fmaf(2.f, x[3], d);                           // x1 - x2 + 2x3
    o[2] = fmaf(4.f, x[3], s);                           // x1 + x2 + 4x3
    o[3] = fmaf(8.f, x[3], d) + x[4];                    // x1 - x2 + 8x3 + x4
  }
};

// F(5,2): points {0, 1, -1, 2, -2, inf}, the point set of F(4,3), so B^T is F(4,3)'s
//   A^T = [1 1 1 1 1 0; 0 1 -1 2 -2 0; 0 1 1 4 4 0; 0 1 -1 8 -8 0; 0 1 1 16 16 1]
constexpr int kAT52[5][6] = {{1, 1, 1, 1, 1, 0}, {0, 1, -1, 2, -2, 0}, {0, 1, 1, 4, 4, 0}, {0, 1, -1, 8, -8, 0},
                             {0, 1, 1, 16, 16, 1}};
static_assert(bt_equal(5, 2, 4, 3) && at_equals<5, 6>(2, kAT52), "F(5,2) tables");
template <>
struct K1<5, 2> {
  static constexpr int L = 6;
  static constexpr bool kPackedBt = true;
  template <typename T>
  __device__ __forceinline__ static void bt(const T (&x)[6], T (&o)[6]) { K1<4, 3>::bt(x, o); }
  __device__ __forceinline__ static void at(const float (&x)[6], float (&o)[5]) {
    const float s1 = x[1] + x[2], d1 = x[1] - x[2], s2 = x[3] + x[4], d2 = x[3] - x[4];
    o[0] = (x[0] + s1) + s2;                             // x0 + x1 + x2 + x3 + x4
    o[1] = fmaf(2.f, d2, d1);                            // x1 - x2 + 2x3 - 2x4
    o[2] = fmaf(4.f, s2, s1);                            // x1 + x2 + 4x3 + 4x4
    o[3] = fmaf(8.f, d2, d1);                            // x1 - x2 + 8x3 - 8x4
    o[4] = fmaf(16.f, s2, s1) + x[5];                    // x1 + x2 + 16x3 + 16x4 + x5
  }
};

// the hand-written F(3,3) / F(4,3) tables above, checked the same way
constexpr int kAT33[3][5] = {{1, 1, 1, 1, 0}, {0, 1, -1, 2, 0}, {0, 1, 1, 4, 1}};
constexpr int kAT43[4][6] = {{1, 1, 1, 1, 1, 0}, {0, 1, -1, 2, -2, 0}, {0, 1, 1, 4, 4, 0}, {0, 1, -1, 8, -8, 1}};
static_assert(at_equals<3, 5>(3, kAT33) && at_equals<4, 6>(3, kAT43), "F(3,3) / F(4,3) output tables");

// ---------------------------------------------------------------------------
// per-axis two-level transforms, float
// ---------------------------------------------------------------------------
// inner level on every reordered column: z[j][p_i] = (B_i^T x[3j .. 3j + l_i))[p_i]
template <int MO, int RO, int MI>
__device__ __forceinline__ void in_axis_inner(const float* x, float (*z)[Ax<MO, RO, MI>::LI]) {
  using X = Ax<MO, RO, MI>;
#pragma unroll
  for (int j = 0; j < X::LO; ++j) {
    float col[X::LI], o[X::LI];
#pragma unroll
    for (int s = 0; s < X::LI; ++s) col[s] = x[kRi * j + s];
    K1<MI, kRi>::bt(col, o);
#pragma unroll
    for (int s = 0; s < X::LI; ++s) z[j][s] = o[s];
  }
}
// outer level for one inner point p_i: o[p_o] = (B_o^T z[.][p_i])[p_o]
template <int MO, int RO, int MI>
__device__ __forceinline__ void in_axis_outer_col(const float (*z)[Ax<MO, RO, MI>::LI], int pi,
                                                  float (&o)[Ax<MO, RO, MI>::LO]) {
  using X = Ax<MO, RO, MI>;
  float c[X::LO];
#pragma unroll
  for (int j = 0; j < X::LO; ++j) c[j] = z[j][pi];
  K1<MO, RO>::bt(c, o);
}

// x[L] (slice window along one axis) -> v[PA] = B^T_hat x, point p = p_o * l_i + p_i
template <int MO, int RO, int MI>
__device__ __forceinline__ void in_axis(const float* x, float* v) {
  using X = Ax<MO, RO, MI>;
  float z[X::LO][X::LI];
  in_axis_inner<MO, RO, MI>(x, z);
#pragma unroll
  for (int pi = 0; pi < X::LI; ++pi) {
    float o[X::LO];
    in_axis_outer_col<MO, RO, MI>(z, pi, o);
#pragma unroll
    for (int po = 0; po < X::LO; ++po) v[po * X::LI + pi] = o[po];
  }
}

// the same three functions on any value type T the 1-D kernels accept (float or f2); packed
// forms exist when both levels' B^T are hand-factored (kPackedAxis)
template <int MO, int RO, int MI>
constexpr bool kPackedAxis = K1<MO, RO>::kPackedBt && K1<MI, kRi>::kPackedBt;
template <int MO, int RO, int MI, typename T>
__device__ __forceinline__ void in_axis_inner_t(const T* x, T (*z)[Ax<MO, RO, MI>::LI]) {
  using X = Ax<MO, RO, MI>;
#pragma unroll
  for (int j = 0; j < X::LO; ++j) {
    T col[X::LI], o[X::LI];
#pragma unroll
    for (int s = 0; s < X::LI; ++s) col[s] = x[kRi * j + s];
    K1<MI, kRi>::bt(col, o);
#pragma unroll
    for (int s = 0; s < X::LI; ++s) z[j][s] = o[s];
  }
}
template <int MO, int RO, int MI, typename T>
__device__ __forceinline__ void in_axis_outer_col_t(const T (*z)[Ax<MO, RO, MI>::LI], int pi,
                                                    T (&o)[Ax<MO, RO, MI>::LO]) {
  using X = Ax<MO, RO, MI>;
  T c[X::LO];
#pragma unroll
  for (int j = 0; j < X::LO; ++j) c[j] = z[j][pi];
  K1<MO, RO>::bt(c, o);
}
template <int MO, int RO, int MI, typename T>
__device__ __forceinline__ void in_axis_t(const T* x, T* v) {
  using X = Ax<MO, RO, MI>;
  T z[X::LO][X::LI];
  in_axis_inner_t<MO, RO, MI, T>(x, z);
#pragma unroll
  for (int pi = 0; pi < X::LI; ++pi) {
    T o[X::LO];
    in_axis_outer_col_t<MO, RO, MI, T>(z, pi, o);
#pragma unroll
    for (int po = 0; po < X::LO; ++po) v[po * X::LI + pi] = o[po];
  }
}

// m[PA] -> y[MA] = A^T_hat m, output q = t * m_i + s
template <int MO, int RO, int MI>
__device__ __forceinline__ void out_axis(const float* m, float* y) {
  using X = Ax<MO, RO, MI>;
  float u[X::LO][MI];
#pragma unroll
  for (int po = 0; po < X::LO; ++po) {
    float col[X::LI], o[MI];
#pragma unroll
    for (int pi = 0; pi < X::LI; ++pi) col[pi] = m[po * X::LI + pi];
    K1<MI, kRi>::at(col, o);
#pragma unroll
    for (int s = 0; s < MI; ++s) u[po][s] = o[s];
  }
#pragma unroll
  for (int s = 0; s < MI; ++s) {
    float col[X::LO], o[MO];
#pragma unroll
    for (int po = 0; po < X::LO; ++po) col[po] = u[po][s];
    K1<MO, RO>::at(col, o);
#pragma unroll
    for (int t = 0; t < MO; ++t) y[t * MI + s] = o[t];
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
