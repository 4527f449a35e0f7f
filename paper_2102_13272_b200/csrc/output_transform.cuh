// output_transform.cuh -- G4: nested output transform fused with the store.
// Instantiated per axis combo in xform_*.cu.
//
// Y = A^T_hat M A_hat per (slice, output channel), then keep mask (redundant
// terms / coverage phases), crop of ragged tiles, depth-to-space of the
// transposed-conv output phases, PReLU and the dtype cast, stored NCHW.
//
// M layout [P][cout_pad][T_pad] fp32.  Persistent kernel, one CTA per SM:
//   warp CO (one elected lane)  TMA producer: one box {32 slices, CO channels,
//                               P_a points} = one point row p_h per ring stage
//   warps 0..CO-1               consumers, warp = output channel, lane = slice
// A unit is (32 consecutive slices, CO channels); its P_a point rows stream
// through an NST-deep ring, so HBM reads stay in flight while the consumers
// compute.  Per point row a consumer applies A^T_hat along w (factored, 25 -> 9,
// compile-time coefficients), accumulates the inner-level A_i^T along h into
// u[m_i][M_a] and, once per outer point p_o, folds u into the output tile with
// A_o^T[t][p_o] (the outer loop is not unrolled, which keeps the kernel inside
// the instruction cache).  The finished tile goes through a per-warp shared
// stage so the stores walk output rows across the 32 slices.
#pragma once
#include <type_traits>

#include "ptx.cuh"
#include "transforms.cuh"

namespace nw {

template <int MO, int RO, int MI, int PRE = 0>
struct OutCfg {
  using X = Ax<MO, RO, MI>;
  // PRE = 1: M already carries the inner output level along w (fused contraction
  // epilogue), so a point row holds l_o * m_i values instead of P_a.  PRE = 2: the inner level
  // is applied along h as well (M''), so a unit has l_o * m_i rows (p_oh, j_h) instead of P_a.
  static constexpr int RL = PRE ? X::LO * MI : X::PA;
  static constexpr int NR = (PRE == 2) ? X::LO * MI : X::PA;   // rows per unit
  // Threads keep (part of) the M_a x M_a output tile in registers.  Up to 9 x 9
  // one thread owns the tile (SPL = 1); larger outer kernels split the output
  // columns by outer index t into SPL parts of TH outer outputs each.
  static constexpr int SPL = (X::MA <= 9) ? 1 : (MO <= 4 ? 2 : 3);
  static constexpr int TH = (MO + SPL - 1) / SPL;   // outer outputs per part
  static constexpr int QW = (SPL == 1) ? X::MA : TH * MI;  // output columns per thread
  // output channels per unit.  Registers are split per SM sub-partition (16K each, warps
  // dealt round-robin): 9 warps allow 168 registers per thread, 13 allow 128.  The
  // kernel is latency-bound, so pre-reduced rows (18 instead of 30 values) buy 12
  // consumer warps for the split 12 x 12 tile.
#ifndef NW_OUT_CO2
#define NW_OUT_CO2 6  // measured: 5 -> +7 %, 7 -> +9 % output-transform time on C2
#endif
  static constexpr int CO = (SPL == 1) ? 8 : (SPL == 2 ? (PRE ? NW_OUT_CO2 : 6) : 3);
  static constexpr int WARPS = CO * SPL;          // consumer warps
  static constexpr int TS = 32;  // slices per unit (lanes)
  static constexpr int STAGE = RL * CO * TS;        // floats per ring stage
  static constexpr int HR = (X::MA + 1) / 2;        // tile rows staged per epilogue phase (two phases)
  // floats per warp output stage; even for column-split tiles, so a warp pair's two stages form
  // one 16-byte-aligned block (the fast store path's [HR][32][12] stage)
  static constexpr int YST = TS * HR * QW + (SPL == 2 ? 2 : 1);
  static constexpr int THREADS = (WARPS + 1) * 32;
  static constexpr size_t YST_BYTES = ((size_t)WARPS * YST * 4 + 127) / 128 * 128;  // keeps sinfo 8-byte aligned
  static constexpr size_t INFO_BYTES = (size_t)WARPS * TS * 16;
  // ring depth (point rows): as deep as shared memory allows, up to 8 -- the kernel streams M
  // at HBM rate only with ~100 KB of loads in flight per SM
  static constexpr size_t FREE = 225 * 1024 - 256 - YST_BYTES - INFO_BYTES;
  static constexpr int NST = (int)(FREE / (STAGE * 4)) > 8 ? 8 : (int)(FREE / (STAGE * 4));
  static constexpr size_t RING_BYTES = (size_t)NST * STAGE * 4;
  static constexpr size_t SMEM = 128 + RING_BYTES + YST_BYTES + INFO_BYTES + 2 * NST * 8;
};

// out_pos / keep as compile-time tables
template <int MO, int RO, int MI>
struct OutTables {
  int pos[kMaxMa];
  unsigned keep[3];  // per coverage phase, bit q
  int shift[3];      // coverage-phase shift
};
template <int MO, int RO, int MI>
__host__ __device__ constexpr OutTables<MO, RO, MI> make_out_tables() {
  OutTables<MO, RO, MI> T{};
  NestedAxis A = make_axis(MO, RO, MI);
  for (int q = 0; q < A.Ma; ++q) T.pos[q] = out_pos(A, q);
  for (int ph = 0; ph < 3; ++ph) {
    unsigned m = 0;
    if (ph < A.nph)
      for (int q = 0; q < A.Ma; ++q)
        if (keep(A, ph, q)) m |= 1u << q;
    T.keep[ph] = m;
    T.shift[ph] = A.shift[ph];
  }
  return T;
}

// v[i] for a runtime i from a compile-time row, as a sum of masked products: a
// select chain gets turned back into an indexed load, which would put the whole
// constexpr coefficient table in local memory
template <int N>
__device__ __forceinline__ float csel(const float (&v)[kMaxL], int i) {
  float r = 0.f;
#pragma unroll
  for (int k = 0; k < N; ++k) {
    if (v[k] != 0.f) r = fmaf((i == k) ? 1.f : 0.f, v[k], r);
  }
  return r;
}

// One unit = 32 slices (lanes) x one output channel coe, one column part: accumulates
// Y = A^T_hat M A_hat from the point rows rowsrc(r, mv) delivers (r = p_o * l_i + p_i),
// then stores the tile (keep mask, crop, depth-to-space, PReLU, cast).
template <int MO, int RO, int MI, typename YT, int PRE, int PART, typename RowSrc>
__device__ __forceinline__ void out_unit(long long t0, int coe, RowSrc&& rowsrc, float* yst, long long* info,
                                         YT* __restrict__ y, const Geometry& g, const float* __restrict__ slopes) {
  using X = Ax<MO, RO, MI>;
  using C = OutCfg<MO, RO, MI, PRE>;
  constexpr AxisF F = axis_f(MO, RO, MI);
  constexpr OutTables<MO, RO, MI> OT = make_out_tables<MO, RO, MI>();
  constexpr int MA = X::MA, LO = X::LO, LI = X::LI, NPH = X::NPH;
  constexpr int RL = C::RL;
  constexpr int QW = C::QW;
  constexpr int T0 = PART * C::TH;                              // first outer output of this part
  const int lane = threadIdx.x & 31;
  const long long HoWo = (long long)g.Ho * g.Wo;
  const int rowstride = (g.mode == 2) ? 2 * g.Wo : g.Wo;
  const int colstride = (g.mode == 2) ? 2 : 1;
  {

    float Y[MA][QW];
#pragma unroll
    for (int i = 0; i < MA; ++i)
#pragma unroll
      for (int j = 0; j < QW; ++j) Y[i][j] = 0.f;

#pragma unroll 1
    for (int p_o = 0; p_o < LO; ++p_o) {
      float uacc[MI][QW];
#pragma unroll
      for (int s = 0; s < MI; ++s)
#pragma unroll
        for (int j = 0; j < QW; ++j) uacc[s][j] = 0.f;
      constexpr int NI = (PRE == 2) ? MI : LI;  // rows per outer point: (p_o, j_h) when the h level is done
#pragma unroll
      for (int p_i = 0; p_i < NI; ++p_i) {
        float mv[RL], qv[QW];
        rowsrc(p_o * NI + p_i, mv);
        // inner level along w on every outer point (done by the contraction epilogue when PRE)
        float uw[LO][MI];
#pragma unroll
        for (int po = 0; po < LO; ++po) {
          if constexpr (PRE) {
#pragma unroll
            for (int s2 = 0; s2 < MI; ++s2) uw[po][s2] = mv[po * MI + s2];
          } else {
            float col[LI], o[MI];
#pragma unroll
            for (int pi = 0; pi < LI; ++pi) col[pi] = mv[po * LI + pi];
            K1<MI, kRi>::at(col, o);
#pragma unroll
            for (int s2 = 0; s2 < MI; ++s2) uw[po][s2] = o[s2];
          }
        }
        if constexpr (C::SPL == 1) {
          // outer level, all outputs
#pragma unroll
          for (int s2 = 0; s2 < MI; ++s2) {
            float col[LO], o[MO];
#pragma unroll
            for (int po = 0; po < LO; ++po) col[po] = uw[po][s2];
            K1<MO, RO>::at(col, o);
#pragma unroll
            for (int t = 0; t < MO; ++t) qv[t * MI + s2] = o[t];
          }
        } else {
          // this part's outer rows (compile-time selection of the F(m_o, r_o) outputs)
#pragma unroll
          for (int s2 = 0; s2 < MI; ++s2) {
            float col[LO], o[MO];
#pragma unroll
            for (int po = 0; po < LO; ++po) col[po] = uw[po][s2];
            K1<MO, RO>::at(col, o);
#pragma unroll
            for (int k = 0; k < C::TH; ++k) qv[k * MI + s2] = (T0 + k < MO) ? o[(T0 + k < MO) ? T0 + k : 0] : 0.f;
          }
        }
        if constexpr (PRE == 2) {
#pragma unroll
          for (int j = 0; j < QW; ++j) uacc[p_i][j] = qv[j];
        } else {
#pragma unroll
        for (int s = 0; s < MI; ++s) {
          const float a = F.AiT[s][p_i];
          if (a == 1.f) {
#pragma unroll
            for (int j = 0; j < QW; ++j) uacc[s][j] += qv[j];
          } else if (a == -1.f) {
#pragma unroll
            for (int j = 0; j < QW; ++j) uacc[s][j] -= qv[j];
          } else if (a != 0.f) {
#pragma unroll
            for (int j = 0; j < QW; ++j) uacc[s][j] = fmaf(a, qv[j], uacc[s][j]);
          }
        }
        }
      }
#pragma unroll
      for (int t = 0; t < MO; ++t) {
        const float c = csel<LO>(F.AoT[t], p_o);
#pragma unroll
        for (int s = 0; s < MI; ++s)
#pragma unroll
          for (int j = 0; j < QW; ++j) Y[t * MI + s][j] = fmaf(c, uacc[s][j], Y[t * MI + s][j]);
      }
    }

    // ---- epilogue: per-slice store geometry (lane = slice), tile -> stage ----
    {
      const long long ts_ = t0 + lane;
      long long b = -1;
      int lim = 0;
      if (ts_ < g.T && coe < g.cout_e) {
        long long tt = ts_;
        const int phw = (int)(tt % NPH);
        tt /= NPH;
        const int phh = (int)(tt % NPH);
        tt /= NPH;
        const int aw = (int)(tt % g.tiles_w);
        tt /= g.tiles_w;
        const int ah = (int)(tt % g.tiles_h);
        const int n = (int)(tt / g.tiles_h);
        int c = coe, fo_h = 0, fo_w = 0;
        if (g.mode == 2) {
          const int f = coe / g.Cout;
          c = coe % g.Cout;
          fo_h = f / 2;
          fo_w = f % 2;
        }
        const int gi0 = ah * X::ADV + (phh == 0 ? OT.shift[0] : phh == 1 ? OT.shift[1] : OT.shift[2]);   // stride-1 grid row of q position 0
        const int gj0 = aw * X::ADV + (phw == 0 ? OT.shift[0] : phw == 1 ? OT.shift[1] : OT.shift[2]);
        int limh, limw;  // positions p with gi0 + p inside the output
        if (g.mode == 2) {
          limh = (g.Ho - fo_h + 1) / 2 - gi0;
          limw = (g.Wo - fo_w + 1) / 2 - gj0;
          b = ((long long)n * g.Cout + c) * HoWo + (long long)(2 * gi0 + fo_h) * g.Wo + (2 * gj0 + fo_w);
        } else {
          limh = g.Hq - gi0;
          limw = g.Wq - gj0;
          b = ((long long)n * g.Cout + c) * HoWo + (long long)gi0 * g.Wo + gj0;
        }
        limh = limh < 0 ? 0 : (limh > 255 ? 255 : limh);
        limw = limw < 0 ? 0 : (limw > 255 ? 255 : limw);
        lim = limh | (limw << 8) | (phh << 16) | (phw << 18);
      }
      info[lane * 2] = b;
      info[lane * 2 + 1] = lim;
    }
    const float slope = (slopes && coe < g.cout_e) ? slopes[g.mode == 2 ? coe % g.Cout : coe] : 0.f;
    // ---- fast store (12 x 12 tiles split over a warp pair, m_i = 3, no depth-to-space, output
    // rows a multiple of 4 wide): the two warps of the channel stage the HR tile rows of all 32
    // slices in one [HR][32 slices][12] block, which is, row by row, the concatenation of the
    // slices' output row segments; each lane then moves 16-byte chunks (3 per row per 32 lanes)
    // with one LDS.128 and one 16-byte (fp32) or 8-byte (bf16) store, instead of one LDS, one
    // STG and the index arithmetic per output.  A chunk never straddles two slices (12 % 4 == 0)
    // and, with Wo % 4 == 0, never straddles the right crop.
    // (fp32 output only: with bf16 y, C3's output transform measured 0.42 -> 0.45 ms on this path;
    // fp32: c2k9 0.133 -> 0.125, c2k5 0.113 -> 0.099, C4a 0.65 -> 0.56, C4b 0.176 -> 0.152 ms,
    // C5 conv1 (fused_c1) 0.85 -> 0.71 ms)
    if constexpr (MI == kRi && C::SPL == 2 && MA == 12 && QW == 6 && C::HR == 6 && 2 * C::YST >= 6 * 32 * 12 &&
                  std::is_same<YT, float>::value) {
      if (g.mode != 2 && g.Wq == g.Wo && (g.Wo & 3) == 0) {
        float* ps = yst - PART * C::YST;                       // the pair's two stages, contiguous
        const int bar_id = 1 + ((int)(threadIdx.x >> 5) >> 1);  // one named barrier per warp pair
        __syncwarp();                                           // info (this warp's copy) written
        long long cb[3];
        int climh[3];
#pragma unroll
        for (int k = 0; k < 3; ++k) {  // chunks q = lane + 32 k of a 384-float stage row
          const int q = lane + 32 * k, sl = q / 3, col = 4 * (q - 3 * sl);
          const long long b = info[sl * 2];
          const int lim = (int)info[sl * 2 + 1];
          const bool ok = b >= 0 && col < ((lim >> 8) & 255);
          cb[k] = ok ? b + col : -1;
          climh[k] = ok ? (lim & 255) : 0;
        }
#pragma unroll
        for (int hph = 0; hph < 2; ++hph) {
#pragma unroll
          for (int i = 0; i < 6; ++i)
#pragma unroll
            for (int j2 = 0; j2 < 3; ++j2)
              *reinterpret_cast<float2*>(ps + (i * 32 + lane) * 12 + PART * 6 + 2 * j2) =
                  make_float2(Y[hph * 6 + i][2 * j2], Y[hph * 6 + i][2 * j2 + 1]);
          asm volatile("bar.sync %0, 64;" ::"r"(bar_id) : "memory");
#pragma unroll
          for (int ii = 0; ii < 3; ++ii) {
            const int i = PART * 3 + ii, qh = hph * 6 + i;
#pragma unroll
            for (int k = 0; k < 3; ++k) {
              float4 v = *reinterpret_cast<const float4*>(ps + i * 384 + 4 * (lane + 32 * k));
              if (qh < climh[k]) {
                if (slopes) {
                  v.x = v.x >= 0.f ? v.x : slope * v.x;
                  v.y = v.y >= 0.f ? v.y : slope * v.y;
                  v.z = v.z >= 0.f ? v.z : slope * v.z;
                  v.w = v.w >= 0.f ? v.w : slope * v.w;
                }
                YT* dst = y + cb[k] + (long long)qh * g.Wo;
                if constexpr (std::is_same<YT, float>::value) {
                  *reinterpret_cast<float4*>(dst) = v;
                } else {
                  __nv_bfloat162 lo2 = __floats2bfloat162_rn(v.x, v.y), hi2 = __floats2bfloat162_rn(v.z, v.w);
                  uint2 u;
                  u.x = *reinterpret_cast<uint32_t*>(&lo2);
                  u.y = *reinterpret_cast<uint32_t*>(&hi2);
                  *reinterpret_cast<uint2*>(dst) = u;
                }
              }
            }
          }
          asm volatile("bar.sync %0, 64;" ::"r"(bar_id) : "memory");  // stage free for the next phase
        }
        return;
      }
    }
    const int qw0 = T0 * MI;  // first output column of this part
    constexpr int HR = C::HR;
    // two phases of HR tile rows each: half the staging buffer, twice the TMA ring depth
#pragma unroll
    for (int hph = 0; hph < 2; ++hph) {
#pragma unroll
      for (int i = 0; i < HR; ++i)
#pragma unroll
        for (int j = 0; j < QW; ++j)
          if (hph * HR + i < MA) yst[lane * (HR * QW) + i * QW + j] = Y[(hph * HR + i < MA) ? hph * HR + i : 0][j];
      __syncwarp();
      // m_i = 3 (no coverage phases): output positions are the identity and every tile
      // output is kept, so only the crop limits are tested per element
      constexpr bool kSimple = (MI == kRi);
#pragma unroll 1
      for (int jj = 0; jj < QW; ++jj) {
        const int e = lane + 32 * jj;  // (slice s, local column ql) pairs, ql fastest
        const int s = e / QW, ql = e - s * QW;
        const int q_w = qw0 + ql;
        const uint32_t ia = ptx::smem_u32(info) + (uint32_t)s * 16u;
        const long long b = ptx::lds_s64(ia);
        const int lim = (int)ptx::lds_s64(ia + 8);
        const uint32_t ya = ptx::smem_u32(yst) + (uint32_t)(s * (HR * QW) + ql) * 4u;
        const int limh = lim & 255, limw = (lim >> 8) & 255;
        unsigned kh = ~0u;
        int pw = q_w;
        bool okw;
        if constexpr (kSimple) {
          okw = b >= 0 && (qw0 + QW <= MA || q_w < MA) && q_w < limw;
        } else {
          const int khi = (lim >> 16) & 3, kwi = (lim >> 18) & 3;
          kh = khi == 0 ? OT.keep[0] : khi == 1 ? OT.keep[1] : OT.keep[2];
          const unsigned kw = kwi == 0 ? OT.keep[0] : kwi == 1 ? OT.keep[1] : OT.keep[2];
          pw = 0;
#pragma unroll
          for (int q = 0; q < MA; ++q) pw = (q_w == q) ? OT.pos[q] : pw;
          okw = b >= 0 && q_w < MA && ((kw >> q_w) & 1u) && pw < limw;
        }
        YT* dst = y + (b < 0 ? 0 : b) + pw * colstride;
        // PReLU and "every tile row inside the image" (warp vote) are resolved once per column
        // group, so the common store is one predicate, one LDS and one STG per element
        auto stores = [&](auto prelu_c, auto rows_in_c) {
          constexpr bool PRELU = decltype(prelu_c)::value, ROWS_IN = decltype(rows_in_c)::value;
#pragma unroll
          for (int i = 0; i < HR; ++i) {
            const int q_h = hph * HR + i;
            const bool kept = kSimple || ((kh >> q_h) & 1u);
            if (q_h < MA && okw && kept && (ROWS_IN || OT.pos[q_h < MA ? q_h : 0] < limh)) {
              float v = ptx::lds_f32(ya + i * QW * 4);
              if constexpr (PRELU) v = v >= 0.f ? v : slope * v;
              dst[OT.pos[q_h < MA ? q_h : 0] * rowstride] = from_f<YT>(v);  // 32-bit row offset
            }
          }
        };
        const bool rows_in = __all_sync(0xffffffffu, limh >= MA);
        if (slopes) {
          if (rows_in) stores(std::true_type{}, std::true_type{});
          else stores(std::true_type{}, std::false_type{});
        } else {
          if (rows_in) stores(std::false_type{}, std::true_type{});
          else stores(std::false_type{}, std::false_type{});
        }
      }
      __syncwarp();
    }
  }
}

template <int MO, int RO, int MI, typename YT, int PRE, int PART>
__device__ __forceinline__ void out_consume(const float* ring, uint64_t* full, uint64_t* empty, float* ystage,
                                            long long* sinfo, YT* __restrict__ y, const Geometry& g,
                                            const float* __restrict__ slopes, int nunits, int ngroups) {
  using C = OutCfg<MO, RO, MI, PRE>;
  constexpr int RL = C::RL;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int cw_ = warp / C::SPL;                                // channel within unit
  float* yst = ystage + warp * C::YST;
  long long* info = sinfo + warp * (C::TS * 2);
  int st = 0;
  uint32_t ph = 0;
  // point rows stream through the TMA ring
  auto ring_row = [&](int, float(&mv)[RL]) {
    ptx::mbar_wait(ptx::smem_u32(&full[st]), ph);
    const float* src = ring + st * C::STAGE + cw_ * C::TS + lane;
#pragma unroll
    for (int p_w = 0; p_w < RL; ++p_w) mv[p_w] = src[p_w * (C::CO * C::TS)];
    __syncwarp();
    if (lane == 0) ptx::mbar_arrive(ptx::smem_u32(&empty[st]));
    if (++st == C::NST) { st = 0; ph ^= 1; }
  };
  for (int u = blockIdx.x; u < nunits; u += gridDim.x) {
    const long long t0 = (long long)(u / ngroups) * C::TS;
    const int coe = (u % ngroups) * C::CO + cw_;
    out_unit<MO, RO, MI, YT, PRE, PART>(t0, coe, ring_row, yst, info, y, g, slopes);
  }
}

template <int MO, int RO, int MI, typename YT, int PRE>
__global__ void __launch_bounds__(OutCfg<MO, RO, MI, PRE>::THREADS, 1)
    output_transform_kernel(const __grid_constant__ CUtensorMap mapM, YT* __restrict__ y, Geometry g,
                            const float* __restrict__ slopes, int nunits, int ngroups) {
  using X = Ax<MO, RO, MI>;
  using C = OutCfg<MO, RO, MI, PRE>;
  constexpr int RL = C::RL;
  constexpr AxisF F = axis_f(MO, RO, MI);
  constexpr OutTables<MO, RO, MI> OT = make_out_tables<MO, RO, MI>();
  constexpr int MA = X::MA, PA = X::PA, LO = X::LO, LI = X::LI, NPH = X::NPH;
  extern __shared__ __align__(128) uint8_t smem_raw[];
  // 128-byte aligned base derived from the shared array itself (keeps loads in the shared window: LDS, not LD)
  uint8_t* base = smem_raw + ((128u - (ptx::smem_u32(smem_raw) & 127u)) & 127u);
  float* ring = reinterpret_cast<float*>(base);
  float* ystage = reinterpret_cast<float*>(base + C::RING_BYTES);
  long long* sinfo = reinterpret_cast<long long*>(base + C::RING_BYTES + C::YST_BYTES);  // [CO][TS][2]
  uint64_t* full = reinterpret_cast<uint64_t*>(base + C::RING_BYTES + C::YST_BYTES + C::INFO_BYTES);
  uint64_t* empty = full + C::NST;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int i = 0; i < C::NST; ++i) {
      ptx::mbar_init(ptx::smem_u32(&full[i]), 1);
      ptx::mbar_init(ptx::smem_u32(&empty[i]), C::WARPS);
    }
    ptx::mbar_init_fence();
  }
  __syncthreads();
  ptx::griddep_launch_dependents();
  ptx::griddep_wait();  // M' / M comes from the contraction just before in the stream

  if (warp == C::WARPS) {
    // ------------------------------ TMA producer ------------------------------
    if (lane == 0) {
      ptx::tma_prefetch(&mapM);
      int st = 0;
      uint32_t ph = 0;
      int waited = -1;  // streamed pipeline: highest 128-slice block whose M' is complete
      for (int u = blockIdx.x; u < nunits; u += gridDim.x) {
        const int t0 = (u / ngroups) * C::TS, co0 = (u % ngroups) * C::CO;
        if (g.sync2) {  // units walk the slices in order: wait for the contraction's units of t0's block
          for (; waited < (t0 >> 7); ++waited) ptx::wait_count(g.sync2 + waited + 1, PA * LO);
        }
        for (int r = 0; r < C::NR; ++r) {
          ptx::mbar_wait(ptx::smem_u32(&empty[st]), ph ^ 1);
          const uint32_t fb = ptx::smem_u32(&full[st]);
          ptx::mbar_expect_tx(fb, C::STAGE * 4);
          ptx::tma_load_3d(ptx::smem_u32(ring + st * C::STAGE), &mapM, fb, t0, co0, r * RL);
          if (++st == C::NST) { st = 0; ph ^= 1; }
        }
      }
    }
    return;
  }

  // -------------------------------- consumers ---------------------------------
  // the column part is a template parameter, so each part's rows of A_o^T are compile-time
  // constants (zero coefficients and unused outputs vanish from the instruction stream)
  const int part = warp % C::SPL;
  if constexpr (C::SPL == 1) {
    out_consume<MO, RO, MI, YT, PRE, 0>(ring, full, empty, ystage, sinfo, y, g, slopes, nunits, ngroups);
  } else if constexpr (C::SPL == 2) {
    if (part == 0) out_consume<MO, RO, MI, YT, PRE, 0>(ring, full, empty, ystage, sinfo, y, g, slopes, nunits, ngroups);
    else out_consume<MO, RO, MI, YT, PRE, 1>(ring, full, empty, ystage, sinfo, y, g, slopes, nunits, ngroups);
  } else {
    if (part == 0) out_consume<MO, RO, MI, YT, PRE, 0>(ring, full, empty, ystage, sinfo, y, g, slopes, nunits, ngroups);
    else if (part == 1) out_consume<MO, RO, MI, YT, PRE, 1>(ring, full, empty, ystage, sinfo, y, g, slopes, nunits, ngroups);
    else out_consume<MO, RO, MI, YT, PRE, 2>(ring, full, empty, ystage, sinfo, y, g, slopes, nunits, ngroups);
  }
}

template <int MO, int RO, int MI, typename YT, int PRE>
static nw_status_t output_launch(const nw_plan_st* p, const Geometry& g, const float* M, void* y, cudaStream_t s) {
  using C = OutCfg<MO, RO, MI, PRE>;
  using X = Ax<MO, RO, MI>;
  auto kern = output_transform_kernel<MO, RO, MI, YT, PRE>;
  if (ensure_smem<output_transform_kernel<MO, RO, MI, YT, PRE>>((int)C::SMEM) != NW_OK) return NW_ERR_CUDA;
  alignas(64) CUtensorMap map;
  const uint64_t rows = PRE ? (uint64_t)C::NR * C::RL : (uint64_t)g.P;
  const uint64_t dims[3] = {(uint64_t)g.T_pad, (uint64_t)g.cout_pad, rows};
  const uint64_t strides[2] = {(uint64_t)g.T_pad * 4, (uint64_t)g.T_pad * g.cout_pad * 4};
  const uint32_t box[3] = {(uint32_t)C::TS, (uint32_t)C::CO, (uint32_t)C::RL};
  if (!encode_tmap(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, M, dims, strides, box, CU_TENSOR_MAP_SWIZZLE_NONE))
    return NW_ERR_CUDA;
  const int ngroups = (g.cout_e + C::CO - 1) / C::CO;  // channel groups holding real channels only
  const long long tchunks = (g.T + C::TS - 1) / C::TS;
  const long long nunits = tchunks * ngroups;
  int sms = 148, dev = 0;
  if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  if (g.ot_ctas > 0 && g.ot_ctas < sms) sms = g.ot_ctas;  // streamed pipeline: its share of the SMs
  const int grid = (int)(nunits < sms ? nunits : sms);
  LaunchScope scope_("output_transform", s);
  if (launch_pdl(kern, dim3(grid), dim3(C::THREADS), C::SMEM, s, map, static_cast<YT*>(y), g,
                 p->prelu ? p->slopes : nullptr, (int)nunits, ngroups) != NW_OK)
    return NW_ERR_CUDA;
  return check_launch();
}

template <int MO, int RO, int MI>
nw_status_t output_impl(const nw_plan_st* p, const Geometry& g, const float* M, void* y, cudaStream_t s) {
  if (p->dtype == NW_DTYPE_BF16) return output_launch<MO, RO, MI, __nv_bfloat16, 0>(p, g, M, y, s);
  return output_launch<MO, RO, MI, float, 0>(p, g, M, y, s);
}
template <int MO, int RO, int MI>
nw_status_t output_impl_pre(const nw_plan_st* p, const Geometry& g, const float* M, void* y, cudaStream_t s) {
  if constexpr (MI == 3) {
    if (p->dtype == NW_DTYPE_BF16) return output_launch<MO, RO, MI, __nv_bfloat16, 1>(p, g, M, y, s);
    return output_launch<MO, RO, MI, float, 1>(p, g, M, y, s);
  }
  return NW_ERR_UNSUPPORTED;
}
template <int MO, int RO, int MI>
nw_status_t output_impl_pre2(const nw_plan_st* p, const Geometry& g, const float* M, void* y, cudaStream_t s) {
  if constexpr (MI == 3) {
    if (p->dtype == NW_DTYPE_BF16) return output_launch<MO, RO, MI, __nv_bfloat16, 2>(p, g, M, y, s);
    return output_launch<MO, RO, MI, float, 2>(p, g, M, y, s);
  }
  return NW_ERR_UNSUPPORTED;
}

}  // namespace nw
