// cooktoom.cuh -- exact (int64 rational) Cook-Toom construction of F(m, r) and
// the composite nested transforms, usable both at compile time (constexpr, so
// the kernels get zero-skipped, constant-folded transforms) and by the host
// planner at run time.
//
// Paper: y = A^T (B^T x (.) G w) (Eq. 2.2); the matrices derive from a
// Vandermonde matrix over interpolation points, which the paper does not
// list (R2: 0, 1, -1, 2, -2, 1/2, -1/2, 4, ..., last point infinity).
// A^T = E_m^T, G = D^-1 E_r, B^T = D Interp^T with D = diag(sgn f_j |f_j|),
// f_j = prod_{i != j}(a_j - a_i): B^T row j = sgn(f_j) coeffs(prod_{i!=j}(x - a_i)),
// G row j = a_j^k / |f_j|; the infinity point contributes the leading
// coefficient (R3).
// Nesting (Eq. 2.5 -> 2.6): per axis the two-level algorithm
// is one bilinear algorithm with B^T_hat = (B_o^T (x) B_i^T) . Gather,
// G_hat = G_o (x) G_i, A^T_hat = A_o^T (x) A_i^T, point index p = p_o*l_i + p_i,
// filter tap k = 3*k1 + k0, output q = t*m_i + s at position 3t + s
// (R4).
#pragma once
#include <cstdint>

namespace nw {

struct Rat {
  long long n = 0, d = 1;
};

__host__ __device__ constexpr long long gcd_ll(long long a, long long b) {
  if (a < 0) a = -a;
  if (b < 0) b = -b;
  while (b) {
    long long t = a % b;
    a = b;
    b = t;
  }
  return a;
}
__host__ __device__ constexpr Rat rat(long long n, long long d = 1) {
  if (d < 0) { n = -n; d = -d; }
  long long g = gcd_ll(n, d);
  if (g == 0) g = 1;
  return Rat{n / g, d / g};
}
__host__ __device__ constexpr Rat radd(Rat a, Rat b) { return rat(a.n * b.d + b.n * a.d, a.d * b.d); }
__host__ __device__ constexpr Rat rsub(Rat a, Rat b) { return rat(a.n * b.d - b.n * a.d, a.d * b.d); }
__host__ __device__ constexpr Rat rmul(Rat a, Rat b) { return rat(a.n * b.n, a.d * b.d); }
__host__ __device__ constexpr Rat rdiv(Rat a, Rat b) { return rat(a.n * b.d, a.d * b.n); }
__host__ __device__ constexpr bool rzero(Rat a) { return a.n == 0; }
__host__ __device__ constexpr double rdouble(Rat a) { return double(a.n) / double(a.d); }

constexpr int kMaxL = 9;   // l = m + r - 1 <= 9 (m <= 6, r <= 4 used here)

struct Kernel1D {
  int m = 0, r = 0, l = 0;
  Rat AT[kMaxL][kMaxL];  // m x l
  Rat G[kMaxL][kMaxL];   // l x r
  Rat BT[kMaxL][kMaxL];  // l x l
};

// k-th finite point in the order 0, 1, -1, 2, -2, 1/2, -1/2, 4, -4, 1/4, ...
__host__ __device__ constexpr Rat point(int k) {
  if (k == 0) return rat(0);
  int j = (k - 1) / 2;            // magnitude index: 1, 2, 1/2, 4, 1/4, ...
  long long num = 1, den = 1;
  if (j > 0) {
    int e = (j + 1) / 2;
    long long p = 1;
    for (int i = 0; i < e; ++i) p *= 2;
    if (j % 2 == 1) num = p; else den = p;
  }
  Rat mag = rat(num, den);
  return (k % 2 == 1) ? mag : rat(-mag.n, mag.d);
}

__host__ __device__ constexpr Kernel1D make_kernel(int m, int r) {
  Kernel1D K{};
  K.m = m; K.r = r; K.l = m + r - 1;
  const int l = K.l;
  const int nfin = (l >= 2) ? l - 1 : 1;   // last point is infinity when l >= 2
  Rat a[kMaxL] = {};
  for (int j = 0; j < nfin; ++j) a[j] = point(j);
  for (int j = 0; j < l; ++j) {
    const bool inf = (l >= 2) && (j == l - 1);
    // polynomial coefficients of prod_{i in S}(x - a_i), S = finite \ {j} (or all)
    Rat c[kMaxL + 1] = {};
    c[0] = rat(1);
    int deg = 0;
    for (int i = 0; i < nfin; ++i) {
      if (!inf && i == j) continue;
      Rat nc[kMaxL + 1] = {};
      for (int t = 0; t <= deg; ++t) {
        nc[t + 1] = radd(nc[t + 1], c[t]);
        nc[t] = rsub(nc[t], rmul(a[i], c[t]));
      }
      ++deg;
      for (int t = 0; t <= deg; ++t) c[t] = nc[t];
    }
    if (inf) {
      for (int i = 0; i < m; ++i) K.AT[i][j] = rat(i == m - 1 ? 1 : 0);
      for (int k = 0; k < r; ++k) K.G[j][k] = rat(k == r - 1 ? 1 : 0);
      for (int t = 0; t < l; ++t) K.BT[j][t] = (t <= deg) ? c[t] : rat(0);
      continue;
    }
    Rat f = rat(1);
    for (int i = 0; i < nfin; ++i)
      if (i != j) f = rmul(f, rsub(a[j], a[i]));
    const bool neg = f.n < 0;
    const Rat af = neg ? rat(-f.n, f.d) : f;
    Rat pw = rat(1);
    for (int i = 0; i < m; ++i) { K.AT[i][j] = pw; pw = rmul(pw, a[j]); }
    pw = rat(1);
    for (int k = 0; k < r; ++k) { K.G[j][k] = rdiv(pw, af); pw = rmul(pw, a[j]); }
    for (int t = 0; t < l; ++t) {
      Rat v = (t <= deg) ? c[t] : rat(0);
      K.BT[j][t] = neg ? rat(-v.n, v.d) : v;
    }
  }
  return K;
}

// Per-axis nested algorithm F(m_o, r_o) (x) F(m_i, 3).
constexpr int kRi = 3;
constexpr int kMaxPa = 64, kMaxLw = 32, kMaxR = 18, kMaxMa = 36;

struct NestedAxis {
  int m_o = 0, r_o = 0, m_i = 0;
  int l_o = 0, l_i = 0, Pa = 0, L = 0, Ma = 0, R = 0;
  int adv = 0, nph = 0;
  int shift[3] = {0, 0, 0};
  Kernel1D ko, ki;
};

__host__ __device__ constexpr NestedAxis make_axis(int m_o, int r_o, int m_i) {
  NestedAxis A{};
  A.m_o = m_o; A.r_o = r_o; A.m_i = m_i;
  A.ko = make_kernel(m_o, r_o);
  A.ki = make_kernel(m_i, kRi);
  A.l_o = A.ko.l; A.l_i = A.ki.l;
  A.Pa = A.l_o * A.l_i;
  A.L = kRi * (A.l_o - 1) + A.l_i;
  A.Ma = m_o * m_i;
  A.R = kRi * r_o;
  if (m_i >= kRi) {                                // contiguous outputs (R5)
    A.nph = 1; A.adv = kRi * (m_o - 1) + m_i;
  } else {                                         // coverage phases (R6)
    A.nph = 0;
    for (int s = 0; s < kRi; s += m_i) A.shift[A.nph++] = s;
    A.adv = kRi * m_o;
  }
  return A;
}

// composite entries (rational)
__host__ __device__ constexpr Rat bt_hat(const NestedAxis& A, int p, int c) {
  const int po = p / A.l_i, pi = p % A.l_i;
  Rat acc = rat(0);
  for (int j = 0; j < A.l_o; ++j) {
    const int s = c - kRi * j;
    if (s >= 0 && s < A.l_i) acc = radd(acc, rmul(A.ko.BT[po][j], A.ki.BT[pi][s]));
  }
  return acc;
}
__host__ __device__ constexpr Rat g_hat(const NestedAxis& A, int p, int k) {
  const int po = p / A.l_i, pi = p % A.l_i, k1 = k / kRi, k0 = k % kRi;
  return rmul(A.ko.G[po][k1], A.ki.G[pi][k0]);
}
__host__ __device__ constexpr Rat at_hat(const NestedAxis& A, int q, int p) {
  const int t = q / A.m_i, s = q % A.m_i, po = p / A.l_i, pi = p % A.l_i;
  return rmul(A.ko.AT[t][po], A.ki.AT[s][pi]);
}
__host__ __device__ constexpr int out_pos(const NestedAxis& A, int q) {
  return kRi * (q / A.m_i) + (q % A.m_i);
}
__host__ __device__ constexpr bool keep(const NestedAxis& A, int phase, int q) {
  const int t = q / A.m_i, s = q % A.m_i;
  if (A.m_i >= kRi) return s < kRi || t == A.m_o - 1;
  return A.shift[phase] + s < kRi;
}

// float copies of the factor matrices for device code
struct AxisF {
  int l_o, l_i, m_o, m_i;
  float BoT[kMaxL][kMaxL], BiT[kMaxL][kMaxL];
  float AoT[kMaxL][kMaxL], AiT[kMaxL][kMaxL];
};
__host__ __device__ constexpr AxisF axis_f(int m_o, int r_o, int m_i) {
  AxisF F{};
  NestedAxis A = make_axis(m_o, r_o, m_i);
  F.l_o = A.l_o; F.l_i = A.l_i; F.m_o = m_o; F.m_i = m_i;
  for (int i = 0; i < kMaxL; ++i)
    for (int j = 0; j < kMaxL; ++j) {
      F.BoT[i][j] = (i < A.l_o && j < A.l_o) ? float(rdouble(A.ko.BT[i][j])) : 0.f;
      F.BiT[i][j] = (i < A.l_i && j < A.l_i) ? float(rdouble(A.ki.BT[i][j])) : 0.f;
      F.AoT[i][j] = (i < A.m_o && j < A.l_o) ? float(rdouble(A.ko.AT[i][j])) : 0.f;
      F.AiT[i][j] = (i < A.m_i && j < A.l_i) ? float(rdouble(A.ki.AT[i][j])) : 0.f;
    }
  return F;
}

}  // namespace nw
