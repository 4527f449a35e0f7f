// input_transform.cuh -- G2: nested input transform V = B^T_hat X B_hat.
// Instantiated per axis combo in xform_*.cu.
//
// Block = (image n, tile row a_h, TW adjacent tiles along w) x CC source
// channels; the channel group is the fastest grid index so the blocks that fill
// one 128-byte V row run together.  256 threads, two passes over shared memory:
//   pass 1  thread = (channel, raw window column): the SR*(shift_max + L) window
//           rows are read straight from x (coalesced along w, zero outside the
//           image = the padding), B^T_hat is applied along h per stride phase
//           p and coverage phase, the P_a results go to Hs[ph][p][p_h][c][col].
//   pass 2  thread = (channel pair, tile, p_h): two L-long rows of Hs are
//           transformed along w; each of the P_a outputs is split into bf16
//           hi/lo (one cvt.rn.bf16x2 per pair and plane) and the pair is stored
//           with one 4-byte store per plane (fp32 path: one 8-byte store).
// A "pair" is two adjacent contraction channels ce: source channels (2k, 2k+1)
// at stride 1, the two column phases q = 0, 1 of one (channel, row phase) at
// stride 2 (ce = 4 ci + 2 p + q, Eq. 2.7 folded into K, R9).
// Channels >= Cin (up to cin_pad) are written as zeros: the contraction runs
// over cin_pad.
#pragma once
#include <cstdlib>

#include "ptx.cuh"
#include "transforms.cuh"

namespace nw {

template <int MO, int RO, int MI, int SR, int CC>
struct InCfg {
  using X = Ax<MO, RO, MI>;
  static constexpr int TW = (X::L <= 17) ? 2 : 1;               // tiles per block along w
  static constexpr int SPAN = (TW - 1) * X::ADV + X::SHMAX + X::L;  // phase-image columns
  static constexpr int WSC = SR * SPAN;                         // raw window columns
  static constexpr int ROWS = SR * (X::SHMAX + X::L);           // raw window rows
  static constexpr int CSTR = WSC | 1;                          // odd channel stride in Hs
  static constexpr int NPAIR = CC * SR * SR / 2;                // ce pairs per block
  static constexpr int PROWS = X::SHMAX + X::L;                 // window rows of one stride phase
  static constexpr int HS = X::NPH * X::PA * CC * CSTR;         // floats (one row phase at a time)
  // stride 2 with 8-channel CTAs (layers with <= 8 source channels, C4a): both row phases' Hs are
  // kept, so pass 2 writes all 4 x cs phase-major contraction channels of a V row at once (full
  // 32-byte sectors; one phase at a time left every sector half written across pass 1 of the
  // other phase, and the L2 re-read the half-written sectors from DRAM: 540 MB of DRAM reads for a
  // 154 MB input, profiles/r2x)
  static constexpr bool BOTH = (SR == 2 && CC == 8);
  // other stride-2 CTAs take one row phase each (twice the CTAs, half the work each): the two
  // phases' window loads are then in flight at once instead of one after the other's pass 2
  static constexpr bool SPLITP = (SR == 2 && !BOTH);
  static constexpr size_t SMEM = (size_t)HS * (BOTH ? 2 : 1) * sizeof(float);
  static constexpr int THREADS = (CC >= 64) ? 512 : (CC >= 32 || SR == 2) ? 256 : 128;
  static constexpr int MINB = 512 / THREADS;                    // resident CTAs per SM (registers <= 128)
};

// Outer level of the w-pass for both channels of a pair, one inner point p_i
// at a time (its l_o outputs share subexpressions), straight into V: points
// p = p_o * l_i + p_i, so the hi / lo pointers walk p_o with stride l_i points
// and p_i with stride one point.
template <int MO, int RO, int MI, bool BF>
__device__ __forceinline__ void store_row(const float (*za)[Ax<MO, RO, MI>::LI], const float (*zb)[Ax<MO, RO, MI>::LI],
                                          char* hp, char* lp, long long stride_bytes) {
  using X = Ax<MO, RO, MI>;
#pragma unroll
  for (int pi = 0; pi < X::LI; ++pi) {
    float oa[X::LO], ob[X::LO];
    in_axis_outer_col<MO, RO, MI>(za, pi, oa);
    in_axis_outer_col<MO, RO, MI>(zb, pi, ob);
    char* h = hp;
    char* l = lp;
#pragma unroll
    for (int po = 0; po < X::LO; ++po) {
      if constexpr (BF) {
        uint32_t hi, lo;
        ptx::split_bf16x2(oa[po], ob[po], hi, lo);
        *reinterpret_cast<uint32_t*>(h) = hi;
        *reinterpret_cast<uint32_t*>(l) = lo;
      } else {
        *reinterpret_cast<float2*>(h) = make_float2(oa[po], ob[po]);
      }
      long long sb = stride_bytes * X::LI;
      asm volatile("" : "+l"(sb));  // incremental pointer walk (no hoisted per-point offsets)
      h += sb;
      if constexpr (BF) l += sb;
    }
    long long sb = stride_bytes;
    asm volatile("" : "+l"(sb));
    hp += sb;
    if constexpr (BF) lp += sb;
  }
}

// Same, for the blocked split layout with a compile-time channel pitch CINP:
// V bytes [T_pad/128][P][2 planes][128 slices][CINP] bf16, so every store of a
// row is the one base pointer plus an immediate (point * 512 * CINP, plane * 256 * CINP).
template <int MO, int RO, int MI, int CINP>
__device__ __forceinline__ void store_row_imm(const float (*za)[Ax<MO, RO, MI>::LI],
                                              const float (*zb)[Ax<MO, RO, MI>::LI], char* hp) {
  using X = Ax<MO, RO, MI>;
  constexpr long long PS = 2ll * 128 * CINP * 2, PL = 128ll * CINP * 2;
#pragma unroll
  for (int pi = 0; pi < X::LI; ++pi) {
    float oa[X::LO], ob[X::LO];
    in_axis_outer_col<MO, RO, MI>(za, pi, oa);
    in_axis_outer_col<MO, RO, MI>(zb, pi, ob);
#pragma unroll
    for (int po = 0; po < X::LO; ++po) {
      uint32_t hi, lo;
      ptx::split_bf16x2(oa[po], ob[po], hi, lo);
      char* h = hp + (po * X::LI + pi) * PS;
      *reinterpret_cast<uint32_t*>(h) = hi;
      *reinterpret_cast<uint32_t*>(h + PL) = lo;
    }
  }
}

// Packed form of store_row_imm: lane 0 of each f2 is channel a, lane 1 channel b; the split's
// subtraction runs on both channels at once (same per-lane rounding as split_bf16x2).
template <int MO, int RO, int MI, int CINP>
__device__ __forceinline__ void store_row_imm_p(const f2 (*zab)[Ax<MO, RO, MI>::LI], char* hp) {
  using X = Ax<MO, RO, MI>;
  constexpr long long PS = 2ll * 128 * CINP * 2, PL = 128ll * CINP * 2;
#pragma unroll
  for (int pi = 0; pi < X::LI; ++pi) {
    f2 o[X::LO];
    in_axis_outer_col_t<MO, RO, MI, f2>(zab, pi, o);
#pragma unroll
    for (int po = 0; po < X::LO; ++po) {
      float a, b;
      f2_unpack(o[po], a, b);
      uint32_t hi, lo;
      asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(hi) : "f"(b), "f"(a));
      const f2 r = o[po] - f2_pack(__uint_as_float(hi << 16), __uint_as_float(hi & 0xffff0000u));
      float ra, rb;
      f2_unpack(r, ra, rb);
      asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(lo) : "f"(rb), "f"(ra));
      char* h = hp + (po * X::LI + pi) * PS;
      *reinterpret_cast<uint32_t*>(h) = hi;
      *reinterpret_cast<uint32_t*>(h + PL) = lo;
    }
  }
}

}  // namespace nw

#include "input_transform_tma.cuh"  // persistent TMA-fed kernel (uses store_row_imm)

namespace nw {

template <int MO, int RO, int MI, int SR, int CC, typename XT, bool BF, int CINP>
__global__ void __launch_bounds__(InCfg<MO, RO, MI, SR, CC>::THREADS, InCfg<MO, RO, MI, SR, CC>::MINB)
    input_transform_kernel(const XT* __restrict__ x, void* __restrict__ Vout,
                                                                 Geometry g, int cgroups, int wgroups) {
  using X = Ax<MO, RO, MI>;
  using C = InCfg<MO, RO, MI, SR, CC>;
  constexpr int PA = X::PA, L = X::L, NPH = X::NPH;
  constexpr int SH1 = X::A.shift[1 < X::A.nph ? 1 : 0];
  extern __shared__ __align__(16) float Hs[];
  const int tid = threadIdx.x;

  int b = blockIdx.x;
  const int pidx = C::SPLITP ? b % 2 : 0;  // SPLITP: this CTA's row phase
  if (C::SPLITP) b /= 2;
  const int cg = b % cgroups;
  b /= cgroups;
  const int wg = b % wgroups;
  b /= wgroups;
  const int ah = b % g.tiles_h;
  const int n = b / g.tiles_h;
  const int cin0 = cg * CC;
  const int aw0 = wg * C::TW;
  const int row0 = SR * (ah * X::ADV) + g.off[0];
  const int col0 = SR * (aw0 * X::ADV) + g.off[0];
  ptx::griddep_launch_dependents();
  ptx::griddep_wait();  // x (and the workspace) may come from the previous kernel in the stream

  const long long pstride = (long long)g.T_pad * g.cin_pad;  // elements between consecutive points
  const long long plane = (long long)g.P * pstride;          // hi -> lo plane (bf16 elements)
  // stride 2: the two row phases p of the polyphase split (Eq. 2.7) run one after the
  // other through the same shared buffer (half the footprint, twice the resident CTAs)
#pragma unroll 1
  for (int p = pidx; p < (C::SPLITP ? pidx + 1 : SR); ++p) {
  if (p > pidx && !C::BOTH) __syncthreads();  // pass 2 of the previous phase is done with Hs
  float* Hp = Hs + (C::BOTH ? p * C::HS : 0);  // this row phase's pass-1 buffer
  // ---------------- pass 1: columns along h (straight from x) ----------------
  // every load of the thread's NT1 columns is issued before the first transform, so a CTA
  // waits for one global round trip per row phase instead of one per column (C2 and, since
  // the interior-window fast path, C3's bf16 x: 0.665 -> 0.587 ms; NW_IN_BATCH_BF16=0 at
  // build time restores the column-at-a-time loop for bf16 x)
#ifndef NW_IN_BATCH_BF16
#define NW_IN_BATCH_BF16 1
#endif
  if constexpr (sizeof(XT) == 4 || NW_IN_BATCH_BF16) {
  constexpr int NT1 = (CC * C::WSC + C::THREADS - 1) / C::THREADS;
  float xr[NT1][C::PROWS];
  const bool rin = row0 + p >= 0 && row0 + p + SR * (C::PROWS - 1) < g.H;
#pragma unroll
  for (int i = 0; i < NT1; ++i) {
    const int task = tid + i * C::THREADS;
    const int col = task % C::WSC, c = task / C::WSC;
    const int ci = cin0 + c, gc = col0 + col;
    const bool cok = task < CC * C::WSC && ci < g.Cin && gc >= 0 && gc < g.W;
    const XT* rp = x + (((long long)n * g.Cin + (cok ? ci : 0)) * g.H) * g.W + (cok ? gc : 0) +
                   (long long)(row0 + p) * g.W;
    if (rin) {  // block-uniform: the whole window column inside the image, no row tests
#pragma unroll
      for (int r = 0; r < C::PROWS; ++r) {
        xr[i][r] = cok ? to_f(*rp) : 0.f;
        long long w = (long long)SR * g.W;
        asm volatile("" : "+l"(w));
        rp += w;
      }
    } else {
#pragma unroll
      for (int r = 0; r < C::PROWS; ++r) {
        const int gr = row0 + p + SR * r;
        xr[i][r] = (cok && gr >= 0 && gr < g.H) ? to_f(*rp) : 0.f;
        long long w = (long long)SR * g.W;
        asm volatile("" : "+l"(w));
        rp += w;
      }
    }
  }
#pragma unroll
  for (int i = 0; i < NT1; ++i) {
    const int task = tid + i * C::THREADS;
    if (task >= CC * C::WSC) break;
    const int col = task % C::WSC, c = task / C::WSC;
#pragma unroll
    for (int ph = 0; ph < NPH; ++ph) {
      const int sh = ph == 0 ? 0 : SH1;
      float xin[L], hv[PA];
#pragma unroll
      for (int r = 0; r < L; ++r) xin[r] = xr[i][sh + r];
      in_axis<MO, RO, MI>(xin, hv);
      float* dst = Hp + (ph * PA * CC + c) * C::CSTR + col;
#pragma unroll
      for (int q = 0; q < PA; ++q) dst[q * CC * C::CSTR] = hv[q];
    }
  }
  } else {
#pragma unroll 1
    for (int task = tid; task < CC * C::WSC; task += C::THREADS) {
      const int col = task % C::WSC, c = task / C::WSC;
      const int ci = cin0 + c, gc = col0 + col;
      const bool cok = ci < g.Cin && gc >= 0 && gc < g.W;
      const XT* rp = x + (((long long)n * g.Cin + (cok ? ci : 0)) * g.H) * g.W + (cok ? gc : 0) +
                     (long long)(row0 + p) * g.W;
      float xc[C::PROWS];
      const bool rin = row0 + p >= 0 && row0 + p + SR * (C::PROWS - 1) < g.H;
#pragma unroll
      for (int r = 0; r < C::PROWS; ++r) {
        const int gr = row0 + p + SR * r;
        xc[r] = (cok && (rin || (gr >= 0 && gr < g.H))) ? to_f(*rp) : 0.f;
        long long w = (long long)SR * g.W;
        asm volatile("" : "+l"(w));
        rp += w;
      }
#pragma unroll
      for (int ph = 0; ph < NPH; ++ph) {
        const int sh = ph == 0 ? 0 : SH1;
        float xin[L], hv[PA];
#pragma unroll
        for (int r = 0; r < L; ++r) xin[r] = xc[sh + r];
        in_axis<MO, RO, MI>(xin, hv);
        float* dst = Hp + (ph * PA * CC + c) * C::CSTR + col;
#pragma unroll
        for (int q = 0; q < PA; ++q) dst[q * CC * C::CSTR] = hv[q];
      }
    }
  }
  if (C::BOTH && p + 1 < SR) continue;  // pass 2 once, after both row phases' pass 1
  __syncthreads();

  // ---------------- pass 2: rows along w, split, store V ----------------
  // channel pairs; stride 2: pairs of each column phase q (phase-major ce = (2p + q) * cs + ci);
  // BOTH: pairs of both row phases, (p, q, channel pair) with the pair fastest, so consecutive
  // lanes write consecutive bytes of a V row
  constexpr int NPR = (SR == 1) ? CC / 2 : (C::BOTH ? 2 * CC : CC);
  constexpr int NTASK = NPH * NPH * PA * C::TW * NPR;
#pragma unroll 1
  for (int task = tid; task < NTASK; task += C::THREADS) {
    int r = task;
    const int pr = r % NPR;
    r /= NPR;
    const int tile = r % C::TW;
    r /= C::TW;
    const int p_h = r % PA;
    r /= PA;
    const int pw = r % NPH;
    const int phh = r / NPH;
    const int aw = aw0 + tile;
    int c0, c1, q0, q1, ce, hoff = 0;
    if (SR == 1) {
      c0 = 2 * pr; c1 = c0 + 1; q0 = q1 = 0;
      ce = cin0 + c0;
    } else {
      const int pb = C::BOTH ? pr / CC : p, prr = C::BOTH ? pr % CC : pr;
      const int q = prr / (CC / 2), cp = prr - q * (CC / 2);
      c0 = 2 * cp; c1 = c0 + 1; q0 = q1 = q;
      ce = (pb * 2 + q) * g.cs + cin0 + c0;
      hoff = C::BOTH ? pb * C::HS : 0;  // row phase pb's pass-1 buffer
    }
    const float* h0 = Hs + hoff + ((phh * PA + p_h) * CC + c0) * C::CSTR;
    const float* h1 = Hs + hoff + ((phh * PA + p_h) * CC + c1) * C::CSTR;
    const int cb = tile * X::ADV + (pw == 0 ? 0 : SH1);
    if (aw >= g.tiles_w || ce >= g.cin_pad || (SR == 2 && cin0 + c0 >= g.cs)) continue;
    float za[X::LO][X::LI], zb[X::LO][X::LI];
    {
      float a[L], bb[L];
#pragma unroll
      for (int k = 0; k < L; ++k) {
        a[k] = h0[SR * (cb + k) + q0];
        bb[k] = h1[SR * (cb + k) + q1];
      }
      in_axis_inner<MO, RO, MI>(a, za);
      in_axis_inner<MO, RO, MI>(bb, zb);
    }
    const long long t = ((((long long)n * g.tiles_h + ah) * g.tiles_w + aw) * NPH + phh) * NPH + pw;
    constexpr int ES = BF ? 2 : 4;
    if (BF && g.vblk) {
      // blocked split layout [T_pad/128][P][hi, lo][128][cin_pad]
      const long long o = ((((t >> 7) * g.P + (long long)p_h * PA) * 2) * 128 + (t & 127)) * g.cin_pad + ce;
      char* hp = reinterpret_cast<char*>(Vout) + o * 2;
      if constexpr (CINP > 0 && BF) {
        store_row_imm<MO, RO, MI, CINP>(za, zb, hp);
      } else {
        store_row<MO, RO, MI, BF>(za, zb, hp, hp + 256ll * g.cin_pad, 512ll * g.cin_pad);
      }
    } else {
      const long long o = ((long long)(p_h * PA) * g.T_pad + t) * g.cin_pad + ce;
      char* hp = reinterpret_cast<char*>(Vout) + o * ES;
      store_row<MO, RO, MI, BF>(za, zb, hp, hp + plane * ES, pstride * ES);
    }
  }
  }  // row phase p
}

template <int MO, int RO, int MI, int SR, int CC, typename XT, bool BF, int CINP>
static nw_status_t input_launch_c(const Geometry& g, const void* x, void* V, cudaStream_t s) {
  using C = InCfg<MO, RO, MI, SR, CC>;
  auto kern = input_transform_kernel<MO, RO, MI, SR, CC, XT, BF, CINP>;
  if (ensure_smem<input_transform_kernel<MO, RO, MI, SR, CC, XT, BF, CINP>>((int)C::SMEM) != NW_OK) return NW_ERR_CUDA;
  const int wgroups = (g.tiles_w + C::TW - 1) / C::TW;
  const int cin_src = (SR == 1) ? g.cin_pad : g.cs;
  const int cgroups = (cin_src + CC - 1) / CC;
  const long long nb = (long long)g.N * g.tiles_h * wgroups * cgroups * (C::SPLITP ? 2 : 1);
  if (nb >= (1ll << 31)) return NW_ERR_UNSUPPORTED;
  LaunchScope scope_("input_transform", s);
  if (launch_pdl(kern, dim3((unsigned)nb), dim3(C::THREADS), C::SMEM, s, static_cast<const XT*>(x), V, g, cgroups,
                 wgroups) != NW_OK)
    return NW_ERR_CUDA;
  return check_launch();
}

// compile-time channel pitch for the common blocked layouts (immediate store offsets)
template <int MO, int RO, int MI, int SR, int CC, typename XT, bool BF>
static nw_status_t input_launch(const Geometry& g, const void* x, void* V, cudaStream_t s) {
  if constexpr (BF && SR == 1 && Ax<MO, RO, MI>::NPH == 1) {  // persistent TMA kernel (input_transform_tma.cuh)
    if (input_tma_eligible<MO, RO, MI, XT>(g)) {
      if (g.cin_pad == 64) return input_tma_launch<MO, RO, MI, XT, 64>(g, x, V, s);
      if (g.cin_pad == 256) return input_tma_launch<MO, RO, MI, XT, 256>(g, x, V, s);
      if (g.cin_pad == 32) return input_tma_launch<MO, RO, MI, XT, 32>(g, x, V, s);
    }
  }
  if (g.sync) return NW_ERR_UNSUPPORTED;  // the streamed pipeline needs the signalling TMA kernel
  if constexpr (BF && SR == 1) {
    if (g.vblk && g.cin_pad == 64) return input_launch_c<MO, RO, MI, SR, CC, XT, BF, 64>(g, x, V, s);
    if (g.vblk && g.cin_pad == 256) return input_launch_c<MO, RO, MI, SR, CC, XT, BF, 256>(g, x, V, s);
    if constexpr (CC == 32)  // C5 deconv (32 source channels)
      if (g.vblk && g.cin_pad == 32) return input_launch_c<MO, RO, MI, SR, CC, XT, BF, 32>(g, x, V, s);
  }
  if constexpr (BF && SR == 2 && sizeof(XT) == 4) {  // C4a (4 x 3 phase channels -> 16), C4b (4 x 64)
    if (g.vblk && g.cin_pad == 16 && CC == 8) return input_launch_c<MO, RO, MI, SR, CC, XT, BF, 16>(g, x, V, s);
    if (g.vblk && g.cin_pad == 256 && CC == 16) return input_launch_c<MO, RO, MI, SR, CC, XT, BF, 256>(g, x, V, s);
  }
  return input_launch_c<MO, RO, MI, SR, CC, XT, BF, 0>(g, x, V, s);
}

template <int MO, int RO, int MI, int SR, typename XT, bool BF>
static nw_status_t input_pick(const Geometry& g, const void* x, void* V, cudaStream_t s) {
  // 16 source channels per 128-thread CTA (4 CTAs / SM), or 32 per 256-thread CTA (2 / SM):
  // NW_IN_CC=32 selects the wide variant where the layer has the channels
  static const int cc = [] {
    const char* v = getenv("NW_IN_CC");
    return v ? atoi(v) : 32;
  }();
  if constexpr (SR == 2) {  // 4 contraction channels per source channel; narrow layers (C4a: 3) take 8-channel CTAs
    if (g.cs <= 8) return input_launch<MO, RO, MI, SR, 8, XT, BF>(g, x, V, s);
    return input_launch<MO, RO, MI, SR, 16, XT, BF>(g, x, V, s);
  } else {
    if constexpr (Ax<MO, RO, MI>::NPH == 1) {
      if (cc >= 64 && g.cin_pad >= 64 && InCfg<MO, RO, MI, SR, 64>::SMEM <= 227 * 1024)
        return input_launch<MO, RO, MI, SR, 64, XT, BF>(g, x, V, s);
      if (cc >= 32 && g.cin_pad >= 32) return input_launch<MO, RO, MI, SR, 32, XT, BF>(g, x, V, s);
    }
    return input_launch<MO, RO, MI, SR, 16, XT, BF>(g, x, V, s);
  }
}

// Instantiated per axis combo in xform_<mo><ro><mi>.cu.  Stride-2 phases and
// bf16 storage are built for the combos the BASELINE configs use.
template <int MO, int RO, int MI>
nw_status_t input_impl(const nw_plan_st* p, const Geometry& g, const void* x, void* V, cudaStream_t s) {
  // stride 2 and bf16 storage are built for the F(m_o,3) (x) F(3,3) plans and the OLA kernel
  constexpr bool kFull = (RO >= 2 && MI == 3 && MO >= 3) || (MO == 1 && RO == 1 && MI == 3);
  constexpr bool kBf16In = kFull || (MO == 2 && RO == 3 && MI == 2);
  const bool bf = p->math != NW_MATH_FP32_SIMT;
  const bool xb = p->dtype == NW_DTYPE_BF16;
  if (g.SR == 1) {
    if (xb) {
      if constexpr (kBf16In) {
        return bf ? input_pick<MO, RO, MI, 1, __nv_bfloat16, true>(g, x, V, s)
                  : input_pick<MO, RO, MI, 1, __nv_bfloat16, false>(g, x, V, s);
      }
      return NW_ERR_UNSUPPORTED;
    }
    return bf ? input_pick<MO, RO, MI, 1, float, true>(g, x, V, s)
              : input_pick<MO, RO, MI, 1, float, false>(g, x, V, s);
  }
  if constexpr (kFull) {
    if (xb)
      return bf ? input_pick<MO, RO, MI, 2, __nv_bfloat16, true>(g, x, V, s)
                : input_pick<MO, RO, MI, 2, __nv_bfloat16, false>(g, x, V, s);
    return bf ? input_pick<MO, RO, MI, 2, float, true>(g, x, V, s)
              : input_pick<MO, RO, MI, 2, float, false>(g, x, V, s);
  }
  return NW_ERR_UNSUPPORTED;
}

}  // namespace nw
