// plan.cu -- the host planner and the host-only half of the C ABI.
//
// The planner restates section IV.B's decomposition for the configurations the
// build supports: a stride-2 layer is split into stride phases
// (Eq. 2.7, "replace F(m, r') by F(m, r'+1) with zero padding") and each
// phase filter longer than 3 taps is nested (III.A) over 3-tap tiles with an
// outer F(m_o, r_o) and inner F(m_i, 3).  The per-phase results are summed in
// the contraction (Cin_e = 4 Cin) -- DESIGN.md#R9.  Transposed stride-2 layers
// use output phases folded into the output channels (R11).
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <new>
#include <vector>

#include "nw_internal.h"

namespace nw {

std::atomic<unsigned long long> g_launches{0};

// Programmatic dependent launch is opt-in (NW_PDL=1): measured 1 % slower on C2 / C3
// (dependent CTAs parked on SMs during the previous kernel's tail), see DESIGN.md section 5.
bool pdl_enabled() {
  static const bool on = [] {
    const char *v = getenv("NW_PDL");
    return v && atoi(v) == 1;
  }();
  return on;
}

static void phase_split(const nw_plan_st *p, int *mode, int *n_sp, int *Kp, int off[2],
                        int taps[2][kMaxTaps]) {
  const int K = p->K;
  for (int a = 0; a < 2; ++a)
    for (int t = 0; t < kMaxTaps; ++t) taps[a][t] = -1;
  if (p->stride == 1) {
    *mode = 0; *n_sp = 1; *Kp = K;
    off[0] = off[1] = -p->pad;
    for (int a = 0; a < K && a < kMaxTaps; ++a) taps[0][a] = a;
    return;
  }
  const int kp = (K + 1) / 2;
  if (!p->transposed) {
    // phase q: y[i] += sum_a x[2(i+a) + q - pad] w[2a + q]   (Eq. 2.7 polyphase)
    *mode = 1; *n_sp = 2; *Kp = kp;
    for (int q = 0; q < 2; ++q) {
      off[q] = q - p->pad;
      for (int a = 0; a < kp; ++a) taps[q][a] = (2 * a + q < K) ? 2 * a + q : -1;
    }
    return;
  }
  // transposed, output phase phi: y[2j + phi] = sum_a x[j + c - a] w[2a + rho],
  // rho = (phi + pad) mod 2, c = (phi + pad - rho)/2; as a correlation over
  // d = kp-1-a the input offset is kp-1-c.  Both phases read one common window
  // (offset omax); the phase with a smaller offset gets leading zero taps.
  *mode = 2; *n_sp = 2;
  int o[2], tl[2][kMaxTaps];
  for (int phi = 0; phi < 2; ++phi) {
    const int rho = (phi + p->pad) % 2;
    const int c = (phi + p->pad - rho) / 2;
    o[phi] = kp - 1 - c;
    for (int d = 0; d < kp; ++d) {
      const int k = 2 * (kp - 1 - d) + rho;
      tl[phi][d] = (k < K) ? k : -1;
    }
  }
  const int omax = o[0] > o[1] ? o[0] : o[1];
  const int omin = o[0] < o[1] ? o[0] : o[1];
  *Kp = kp + omax - omin;
  for (int phi = 0; phi < 2; ++phi) {
    const int lead = omax - o[phi];
    for (int d = 0; d < *Kp && d < kMaxTaps; ++d) {
      const int s = d - lead;
      taps[phi][d] = (s >= 0 && s < kp) ? tl[phi][s] : -1;
    }
    off[phi] = omax;  // stored positive here; Geometry negates
  }
}

nw_status_t finalize(nw_plan_st *p) {
  if (p->finalized) return NW_OK;
  if (p->pad < 0) p->pad = p->K / 2;
  if (p->transposed && p->stride != 2) return NW_ERR_UNSUPPORTED;
  if (p->depthwise) {  // groups = C: one filter per channel, no channel sum
    if (p->Cin != p->Cout) return NW_ERR_INVALID;
    if (p->stride != 1 || p->transposed || p->math == NW_MATH_BF16) return NW_ERR_UNSUPPORTED;
  }
  int mode, n_sp, Kp, off[2], taps[2][kMaxTaps];
  phase_split(p, &mode, &n_sp, &Kp, off, taps);
  p->Kp = Kp;
  p->r_o = p->outer_taps ? p->outer_taps : (Kp + 2) / 3;
  if (p->r_o < 1 || p->r_o > 6) return NW_ERR_INVALID;
  if (Kp > 3 * p->r_o) return NW_ERR_UNSUPPORTED;
  if (p->m_o + p->r_o - 1 > kMaxL || p->m_i + 2 > kMaxL) return NW_ERR_UNSUPPORTED;
  p->ax = make_axis(p->m_o, p->r_o, p->m_i);
  p->cin_e = p->Cin * ((mode == 1) ? 4 : 1);
  p->cout_e = p->Cout * ((mode == 2) ? 4 : 1);
  // stride 2: contraction channels are phase-major, ce = (2p + q) * cs + ci, with the per-phase
  // stride cs = Cin rounded up to a multiple of 4: channel pairs never straddle two phases and
  // 4 cs is already a multiple of the 16-channel granule (every channel is written)
  p->cs = (mode == 1) ? (int)round_up(p->Cin, 4) : p->Cin;
  p->cin_pad = (int)round_up((mode == 1) ? 4 * p->cs : p->cin_e, kGranule);
  p->cout_pad = (int)round_up(p->cout_e, kGranule);
  if (p->prelu && !p->slopes) return NW_ERR_INVALID;
  p->finalized = true;
  return NW_OK;
}

NestedAxis path_axis(const nw_plan_st *p, int path) {
  if (path == kPathNested) return p->ax;
  if (path == kPathOla) return make_axis(1, 1, kRi);  // single-level F(3,3) = F(1,1) (x) F(3,3)
  NestedAxis A{};                                      // direct: no transform, one point, pixel tiles
  A.m_o = A.r_o = A.m_i = 1;
  A.l_o = A.l_i = A.Pa = A.L = A.Ma = A.R = 1;
  A.adv = 1;
  A.nph = 1;
  return A;
}

// Slice geometry of one path.  Nested: slices of adv x adv outputs.
// OLA (Eq. 2.3): 3x3-output F(3,3) tiles; the nb x nb filter blocks read the
// tile grid shifted by (bh, bw), so the grid is extended by nb - 1 tiles per
// axis and block b's operand is V row t + bh * tiles_w + bw.  Direct (Eq. 2.1):
// one "tile" per pixel of the (phase) input grid extended by Kp - 1; tap
// (a, b) reads pixel row t + a * tiles_w + b.
Geometry make_geometry(const nw_plan_st *p, int N, int H, int W, int path) {
  Geometry g{};
  int off[2];
  phase_split(p, &g.mode, &g.n_sp, &g.Kp, off, g.taps);
  g.SR = (g.mode == 1) ? 2 : 1;
  for (int a = 0; a < 2; ++a) g.off[a] = (g.mode == 2) ? -off[a] : off[a];
  const NestedAxis ax = path_axis(p, path);
  g.path = path;
  g.adv = ax.adv;
  g.nph = ax.nph;
  for (int i = 0; i < 3; ++i) g.shift[i] = ax.shift[i];
  g.N = N; g.Cin = p->Cin; g.Cout = p->Cout; g.H = H; g.W = W;
  if (g.mode == 2) {
    g.Ho = (H - 1) * 2 - 2 * p->pad + p->K + p->output_padding;
    g.Wo = (W - 1) * 2 - 2 * p->pad + p->K + p->output_padding;
    g.Hq = (g.Ho + 1) / 2;
    g.Wq = (g.Wo + 1) / 2;
  } else {
    g.Ho = (H + 2 * p->pad - p->K) / p->stride + 1;
    g.Wo = (W + 2 * p->pad - p->K) / p->stride + 1;
    g.Hq = g.Ho;
    g.Wq = g.Wo;
  }
  g.tiles_h = (g.Hq + g.adv - 1) / g.adv;
  g.tiles_w = (g.Wq + g.adv - 1) / g.adv;
  if (path == kPathNested) {
    g.mo = p->m_o; g.ro = p->r_o; g.mi = p->m_i;
    g.R = kRi * p->r_o;
    g.nb = 1;
  } else if (path == kPathOla) {
    g.mo = 1; g.ro = 1; g.mi = kRi;
    g.R = kRi;
    g.nb = (g.Kp + kRi - 1) / kRi;
  } else {
    g.mo = g.ro = g.mi = 1;
    g.R = 1;
    g.nb = g.Kp;
  }
  g.tiles_h += g.nb - 1;
  g.tiles_w += g.nb - 1;
  g.nsh = g.nb * g.nb;
  g.T = (long long)N * g.tiles_h * g.tiles_w * g.nph * g.nph;
  g.T_pad = round_up(g.T, 128);
  g.cin_e = p->cin_e; g.cout_e = p->cout_e;
  g.cs = p->cs;
  g.cin_pad = p->cin_pad; g.cout_pad = p->cout_pad;
  g.Pa = ax.Pa;
  g.P = g.Pa * g.Pa;
  g.vblk = (path == kPathNested && p->math == NW_MATH_BF16X3) ? 1 : 0;
  return g;
}

size_t v_bytes(const nw_plan_st *p, const Geometry &g) {
  // fp32, or two bf16 planes (hi, lo): 4 bytes per element either way
  (void)p;
  return (size_t)round_up((long long)g.P * g.T_pad * g.cin_pad * 4, 256);
}
size_t m_bytes(const nw_plan_st *p, const Geometry &g) {
  (void)p;
  return (size_t)round_up((long long)g.P * g.T_pad * g.cout_pad * 4, 256);
}
size_t u_bytes(const Geometry &g) {
  return (size_t)round_up((long long)g.P * g.cout_pad * g.nsh * g.cin_pad * 4, 256);
}
size_t filter_bytes(const nw_plan_st *p) {
  const long long P = (long long)p->ax.Pa * p->ax.Pa;
  if (p->depthwise) return (size_t)(P * p->cout_pad * 4);  // fp32 U [P][cout_pad]: one filter per channel
  return (size_t)(P * p->cout_pad * p->cin_pad * 4);  // fp32 or bf16 hi + lo planes
}

}  // namespace nw

using namespace nw;

extern "C" {

const char *nw_status_str(nw_status_t s) {
  switch (s) {
    case NW_OK: return "ok";
    case NW_ERR_INVALID: return "invalid argument";
    case NW_ERR_UNSUPPORTED: return "unsupported configuration";
    case NW_ERR_NOMEM: return "out of host memory";
    case NW_ERR_CUDA: return "CUDA error";
    case NW_ERR_WORKSPACE: return "workspace too small";
    case NW_ERR_STATE: return "plan already finalized";
  }
  return "unknown status";
}

unsigned long long nw_launch_count(void) { return g_launches.load(); }

nw_status_t nw_plan(int K, int stride, int m_outer, int m_inner, int Cin, int Cout, nw_plan_t *out) {
  if (!out) return NW_ERR_INVALID;
  *out = nullptr;
  if (K < 1 || Cin < 1 || Cout < 1) return NW_ERR_INVALID;
  if (m_outer < 1 || m_outer > 6 || m_inner < 1 || m_inner > 6) return NW_ERR_INVALID;
  if (stride != 1 && stride != 2) return NW_ERR_UNSUPPORTED;
  if (K > 9 * stride) return NW_ERR_UNSUPPORTED;
  nw_plan_st *p = new (std::nothrow) nw_plan_st();
  if (!p) return NW_ERR_NOMEM;
  p->K = K; p->stride = stride; p->m_o = m_outer; p->m_i = m_inner; p->Cin = Cin; p->Cout = Cout;
  *out = p;
  return NW_OK;
}

nw_status_t nw_plan_set(nw_plan_t p, nw_attr_t attr, long long v) {
  if (!p) return NW_ERR_INVALID;
  if (p->finalized) return NW_ERR_STATE;
  switch (attr) {
    case NW_ATTR_MATH:
      if (v < NW_MATH_FP32_SIMT || v > NW_MATH_BF16) return NW_ERR_INVALID;
      p->math = (int)v; return NW_OK;
    case NW_ATTR_DTYPE:
      if (v != NW_DTYPE_F32 && v != NW_DTYPE_BF16) return NW_ERR_INVALID;
      p->dtype = (int)v; return NW_OK;
    case NW_ATTR_TRANSPOSED:
      if (v != 0 && v != 1) return NW_ERR_INVALID;
      if (v && p->stride != 2) return NW_ERR_UNSUPPORTED;
      p->transposed = (int)v; return NW_OK;
    case NW_ATTR_OUTPUT_PADDING:
      if (v < 0 || v > 1) return NW_ERR_INVALID;
      p->output_padding = (int)v; return NW_OK;
    case NW_ATTR_OUTER_TAPS:
      if (v < 0 || v > 6) return NW_ERR_INVALID;
      p->outer_taps = (int)v; return NW_OK;
    case NW_ATTR_PAD:
      if (v < 0 || v > 64) return NW_ERR_INVALID;
      p->pad = (int)v; return NW_OK;
    case NW_ATTR_PRELU:
      if (v != 0 && v != 1) return NW_ERR_INVALID;
      p->prelu = (int)v; return NW_OK;
    case NW_ATTR_DEPTHWISE:
      if (v != 0 && v != 1) return NW_ERR_INVALID;
      p->depthwise = (int)v; return NW_OK;
  }
  return NW_ERR_INVALID;
}

nw_status_t nw_plan_set_prelu(nw_plan_t p, const float *slopes) {
  if (!p || !slopes) return NW_ERR_INVALID;
  if (p->finalized) return NW_ERR_STATE;
  p->slopes = slopes;
  p->prelu = 1;
  return NW_OK;
}

nw_status_t nw_plan_finalize(nw_plan_t p) {
  if (!p) return NW_ERR_INVALID;
  return finalize(p);
}

nw_status_t nw_plan_destroy(nw_plan_t p) {
  if (!p) return NW_ERR_INVALID;
  delete p;
  return NW_OK;
}

nw_status_t nw_plan_info(nw_plan_t p, nw_plan_info_t *info) {
  if (!p || !info) return NW_ERR_INVALID;
  nw_status_t st = finalize(p);
  if (st != NW_OK) return st;
  std::memset(info, 0, sizeof(*info));
  info->K = p->K; info->stride = p->stride; info->transposed = p->transposed;
  info->pad = p->pad; info->output_padding = p->output_padding;
  info->m_outer = p->m_o; info->r_outer = p->r_o; info->m_inner = p->m_i;
  info->points_axis = p->ax.Pa;
  info->points = p->ax.Pa * p->ax.Pa;
  info->window = p->ax.L;
  info->tile_out = p->ax.adv;
  info->n_phase = p->ax.nph;
  info->Kp = p->Kp;
  info->cin = p->Cin; info->cout = p->Cout;
  info->cin_e = p->cin_e; info->cout_e = p->cout_e;
  info->cin_pad = p->cin_pad; info->cout_pad = p->cout_pad;
  info->math = p->math; info->dtype = p->dtype;
  info->filter_bytes = filter_bytes(p);
  {
    // a representative geometry: 16-byte x rows (the single-kernel paths load x by TMA)
    const int side = (int)round_up(3 * p->K + 16, 8);
    Geometry g = make_geometry(p, 1, side, side);
    const int fl = gemm_fused_level(p, g);
    info->m_rows = fl == 2 ? (p->ax.l_o * p->m_i) * (p->ax.l_o * p->m_i)
                           : (fl == 1 ? p->ax.Pa * p->ax.l_o * p->m_i : info->points);
    info->single_kernel = (fused_c1_eligible(p, g) || fused_co_eligible(p, g)) ? 1 : 0;
    if (info->single_kernel) info->m_rows = 0;
  }
  return NW_OK;
}

nw_status_t nw_plan_tables(nw_plan_t p, int which, long long *dst, size_t cap, size_t *n) {
  if (!p || !n) return NW_ERR_INVALID;
  nw_status_t st = finalize(p);
  if (st != NW_OK) return st;
  const NestedAxis &A = p->ax;
  std::vector<long long> t;
  auto push_rat = [&](Rat r) { t.push_back(r.n); t.push_back(r.d); };
  switch (which) {
    case NW_TABLE_BT:
      for (int q = 0; q < A.Pa; ++q)
        for (int c = 0; c < A.L; ++c) push_rat(bt_hat(A, q, c));
      break;
    case NW_TABLE_G:
      for (int q = 0; q < A.Pa; ++q)
        for (int k = 0; k < A.R; ++k) push_rat(g_hat(A, q, k));
      break;
    case NW_TABLE_AT:
      for (int q = 0; q < A.Ma; ++q)
        for (int c = 0; c < A.Pa; ++c) push_rat(at_hat(A, q, c));
      break;
    case NW_TABLE_GATHER:
      for (int j = 0; j < A.l_o; ++j)
        for (int s = 0; s < A.l_i; ++s) t.push_back(kRi * j + s);
      break;
    case NW_TABLE_SCATTER:
      for (int ph = 0; ph < A.nph; ++ph)
        for (int q = 0; q < A.Ma; ++q) {
          t.push_back(A.shift[ph] + out_pos(A, q));
          t.push_back(keep(A, ph, q) ? 1 : 0);
        }
      break;
    case NW_TABLE_ORIGINS:
      t.push_back(A.adv);
      t.push_back(A.nph);
      for (int ph = 0; ph < A.nph; ++ph) t.push_back(A.shift[ph]);
      break;
    case NW_TABLE_PHASE_TAPS: {
      int mode, n_sp, Kp, off[2], taps[2][kMaxTaps];
      phase_split(p, &mode, &n_sp, &Kp, off, taps);
      t.push_back(mode);
      t.push_back(n_sp);
      t.push_back(Kp);
      for (int ph = 0; ph < n_sp; ++ph) {
        t.push_back(mode == 0 ? -off[ph] : off[ph]);  // mode 0: pad; mode 1: p - pad; mode 2: offset
        for (int a = 0; a < Kp; ++a) t.push_back(taps[ph][a]);
      }
      break;
    }
    case NW_TABLE_DIMS: {
      const long long v[] = {p->K, p->stride, p->transposed, p->m_o, p->r_o, p->m_i, A.l_o, A.l_i, A.Pa,
                             A.L, A.Ma, (long long)A.Pa * A.Pa, p->Cin, p->Cout, p->cin_e, p->cout_e,
                             p->Kp, A.nph, A.adv};
      t.assign(v, v + sizeof(v) / sizeof(v[0]));
      break;
    }
    default:
      return NW_ERR_INVALID;
  }
  *n = t.size();
  if (cap == 0 && !dst) return NW_OK;
  if (!dst || cap < t.size()) return NW_ERR_INVALID;
  std::memcpy(dst, t.data(), t.size() * sizeof(long long));
  return NW_OK;
}

nw_status_t nw_output_size(nw_plan_t p, int H, int W, int *Ho, int *Wo) {
  if (!p || !Ho || !Wo || H < 1 || W < 1) return NW_ERR_INVALID;
  nw_status_t st = finalize(p);
  if (st != NW_OK) return st;
  Geometry g = make_geometry(p, 1, H, W);
  if (g.Ho < 1 || g.Wo < 1) return NW_ERR_INVALID;
  *Ho = g.Ho;
  *Wo = g.Wo;
  return NW_OK;
}

nw_status_t nw_workspace_size(nw_plan_t p, int N, int H, int W, size_t *bytes) {
  if (!p || !bytes || N < 1 || H < 1 || W < 1) return NW_ERR_INVALID;
  nw_status_t st = finalize(p);
  if (st != NW_OK) return st;
  Geometry g = make_geometry(p, N, H, W);
  if (g.Ho < 1 || g.Wo < 1) return NW_ERR_INVALID;
  *bytes = forward_ws_bytes(p, N, H, W);
  return NW_OK;
}

nw_status_t nw_count_mults(nw_plan_t p, int N, int H, int W, unsigned long long *ewmm) {
  if (!p || !ewmm || N < 1 || H < 1 || W < 1) return NW_ERR_INVALID;
  nw_status_t st = finalize(p);
  if (st != NW_OK) return st;
  Geometry g = make_geometry(p, N, H, W);
  // depthwise: one product per (slice, point, channel) -- no channel contraction
  *ewmm = (unsigned long long)g.T * g.P * (p->depthwise ? (unsigned long long)g.cout_e
                                                         : (unsigned long long)g.cin_e * g.cout_e);
  return NW_OK;
}

}  // extern "C"
