// input_transform.cuh -- G2 kernel template (instantiated per axis combo in input_*.cu)
#pragma once
#include "transforms.cuh"

namespace nw {

// ---------------------------------------------------------------------------
// G2: input transform
// Block = (n, tile row a_h, TW tiles along w) x CC input channels.  The input
// region (rows of every coverage / stride phase, TW slice windows) is staged in
// shared memory [row][col][cc] (zero-filled outside the image = the padding).
// Pass 1 transforms every staged column along h (B^T_hat on rows) into
// Hs[p_h][col][cc]; pass 2 transforms along w per (tile, p_h) and stores the
// P_a values of V[xi = p_h*P_a + p_w][t][ce].  With bf16 output each lane pair
// exchanges (hi, lo) so one lane writes the hi plane pair and the other the lo
// plane pair (4-byte stores, full 32-byte sectors per 8 lanes).
// ---------------------------------------------------------------------------
template <int MO, int RO, int MI, int SR>
struct InCfg {
  using X = Ax<MO, RO, MI>;
  static constexpr int CC = (SR == 1) ? 16 : 8;
  static constexpr int TW = 2;
  static constexpr int SPAN = (TW - 1) * X::ADV + X::SHMAX + X::L;
  static constexpr int WSC = SR * SPAN;
  static constexpr int ROWS = SR * (X::SHMAX + X::L);
  static constexpr int CCP = CC + 1;
  static constexpr int HCC = CC;
  static constexpr int XS = ROWS * WSC * CCP;
  static constexpr int HS = X::PA * WSC * HCC;
  static constexpr size_t SMEM = (size_t)(XS + HS) * sizeof(float);
};

template <int MO, int RO, int MI, int SR, typename XT, bool BF>
__global__ void __launch_bounds__(256) input_transform_kernel(const XT* __restrict__ x, void* __restrict__ Vout,
                                                              Geometry g) {
  using X = Ax<MO, RO, MI>;
  using C = InCfg<MO, RO, MI, SR>;
  constexpr int SHIFT[3] = {X::A.shift[0], X::A.shift[1], X::A.shift[2]};
  extern __shared__ __align__(16) float smem[];
  float* Xs = smem;
  float* Hs = smem + C::XS;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wgroups = (g.tiles_w + C::TW - 1) / C::TW;
  int b = blockIdx.x;
  const int wg = b % wgroups;
  b /= wgroups;
  const int ah = b % g.tiles_h;
  const int n = b / g.tiles_h;
  const int cin0 = blockIdx.y * C::CC;
  const int aw0 = wg * C::TW;
  const int row0 = SR * (ah * X::ADV) + g.off[0];
  const int col0 = SR * (aw0 * X::ADV) + g.off[0];

  // stage the input region (coalesced along w, zero outside = padding)
  for (int idx = tid; idx < C::CC * C::ROWS * C::WSC; idx += blockDim.x) {
    const int c = idx % C::WSC;
    const int r = (idx / C::WSC) % C::ROWS;
    const int cc = idx / (C::WSC * C::ROWS);
    const int gr = row0 + r, gc = col0 + c, ci = cin0 + cc;
    float v = 0.f;
    if (ci < g.Cin && gr >= 0 && gr < g.H && gc >= 0 && gc < g.W)
      v = to_f(x[(((long long)n * g.Cin + ci) * g.H + gr) * g.W + gc]);
    Xs[(r * C::WSC + c) * C::CCP + cc] = v;
  }

  const long long plane = (long long)g.P * g.T_pad * g.cin_pad;
#pragma unroll
  for (int ph = 0; ph < X::NPH; ++ph) {
#pragma unroll
    for (int p = 0; p < SR; ++p) {
      __syncthreads();
      // pass 1: columns along h
      for (int task = tid; task < C::CC * C::WSC; task += blockDim.x) {
        const int cc = task % C::CC, col = task / C::CC;
        float xin[X::L], hv[X::PA];
#pragma unroll
        for (int r = 0; r < X::L; ++r)
          xin[r] = Xs[((SR * (SHIFT[ph] + r) + p) * C::WSC + col) * C::CCP + cc];
        in_axis<MO, RO, MI>(xin, hv);
#pragma unroll
        for (int q = 0; q < X::PA; ++q) Hs[(q * C::WSC + col) * C::HCC + cc] = hv[q];
      }
      __syncthreads();
      // pass 2: rows along w, store V
      constexpr int NTASK = SR * C::CC * C::TW * X::PA;  // multiple of 32
#pragma unroll
      for (int pw = 0; pw < X::NPH; ++pw) {
        for (int base = warp * 32; base < NTASK; base += blockDim.x) {
          const int task = base + lane;
          const int q = task % SR;
          int rest = task / SR;
          const int cc = rest % C::CC;
          rest /= C::CC;
          const int tile = rest % C::TW;
          const int p_h = rest / C::TW;
          const int aw = aw0 + tile;
          const int ci = cin0 + cc;
          const int ce = (SR == 1) ? ci : ci * 4 + p * 2 + q;
          const bool valid = (aw < g.tiles_w) && (ce < g.cin_pad);
          float hin[X::L], vv[X::PA];
#pragma unroll
          for (int c = 0; c < X::L; ++c)
            hin[c] = Hs[(p_h * C::WSC + SR * (tile * X::ADV + SHIFT[pw] + c) + q) * C::HCC + cc];
          in_axis<MO, RO, MI>(hin, vv);
          const long long t = ((((long long)n * g.tiles_h + ah) * g.tiles_w + aw) * X::NPH + ph) * X::NPH + pw;
#pragma unroll
          for (int p_w = 0; p_w < X::PA; ++p_w) {
            const long long o = ((long long)(p_h * X::PA + p_w) * g.T_pad + t) * g.cin_pad + ce;
            if (BF) {
              const float v = vv[p_w];
              const __nv_bfloat16 hi = __float2bfloat16_rn(v);
              const __nv_bfloat16 lo = __float2bfloat16_rn(v - __bfloat162float(hi));
              const unsigned mine = (unsigned)__bfloat16_as_ushort(hi) | ((unsigned)__bfloat16_as_ushort(lo) << 16);
              const unsigned other = __shfl_xor_sync(0xffffffffu, mine, 1);
              if (valid) {
                __nv_bfloat16* V = reinterpret_cast<__nv_bfloat16*>(Vout);
                if ((lane & 1) == 0) {
                  *reinterpret_cast<unsigned*>(V + o) = (mine & 0xffffu) | (other << 16);
                } else {
                  *reinterpret_cast<unsigned*>(V + plane + o - 1) = (other >> 16) | (mine & 0xffff0000u);
                }
              }
            } else if (valid) {
              reinterpret_cast<float*>(Vout)[o] = vv[p_w];
            }
          }
        }
      }
    }
  }
}

}  // namespace nw

namespace nw {

template <int MO, int RO, int MI, int SR, typename XT, bool BF>
static nw_status_t input_launch(const Geometry& g, const void* x, void* V, cudaStream_t s) {
  using C = InCfg<MO, RO, MI, SR>;
  auto kern = input_transform_kernel<MO, RO, MI, SR, XT, BF>;
  static bool attr_done = false;  // per instantiation
  if (!attr_done) {
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::SMEM) != cudaSuccess)
      return NW_ERR_CUDA;
    attr_done = true;
  }
  const int wgroups = (g.tiles_w + C::TW - 1) / C::TW;
  const long long gx = (long long)g.N * g.tiles_h * wgroups;
  const int cin_src = (SR == 1) ? g.cin_pad : g.cin_pad / 4;
  dim3 grid((unsigned)gx, (unsigned)((cin_src + C::CC - 1) / C::CC));
  LaunchScope scope_("input_transform", s);
  kern<<<grid, 256, C::SMEM, s>>>(static_cast<const XT*>(x), V, g);
  return check_launch();
}

// Instantiated per axis combo in input_<mo><ro><mi>.cu.  Stride-2 phases and
// bf16 storage are built for the combos the BASELINE configs use.
template <int MO, int RO, int MI>
nw_status_t input_impl(const nw_plan_st* p, const Geometry& g, const void* x, void* V, cudaStream_t s) {
  constexpr bool kFull = (MO == 3 && RO == 3 && MI == 3);
  constexpr bool kBf16In = kFull || (MO == 2 && RO == 3 && MI == 2);
  const bool bf = p->math != NW_MATH_FP32_SIMT;
  const bool xb = p->dtype == NW_DTYPE_BF16;
  if (g.SR == 1) {
    if (xb) {
      if constexpr (kBf16In) {
        return bf ? input_launch<MO, RO, MI, 1, __nv_bfloat16, true>(g, x, V, s)
                  : input_launch<MO, RO, MI, 1, __nv_bfloat16, false>(g, x, V, s);
      }
      return NW_ERR_UNSUPPORTED;
    }
    return bf ? input_launch<MO, RO, MI, 1, float, true>(g, x, V, s)
              : input_launch<MO, RO, MI, 1, float, false>(g, x, V, s);
  }
  if constexpr (kFull) {
    if (xb)
      return bf ? input_launch<MO, RO, MI, 2, __nv_bfloat16, true>(g, x, V, s)
                : input_launch<MO, RO, MI, 2, __nv_bfloat16, false>(g, x, V, s);
    return bf ? input_launch<MO, RO, MI, 2, float, true>(g, x, V, s)
              : input_launch<MO, RO, MI, 2, float, false>(g, x, V, s);
  }
  return NW_ERR_UNSUPPORTED;
}

}  // namespace nw
