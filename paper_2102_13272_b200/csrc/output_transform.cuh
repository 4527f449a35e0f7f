// output_transform.cuh -- G4 kernel template (instantiated per axis combo in output_*.cu)
#pragma once
#include "transforms.cuh"

namespace nw {

// ---------------------------------------------------------------------------
// G4: output transform + keep/crop + (depth-to-space) + PReLU + store
// Block = (n, a_h, TWO tiles along w) x CO output channels (of Cout_e).
// ---------------------------------------------------------------------------
template <int MO, int RO, int MI>
struct OutCfg {
  using X = Ax<MO, RO, MI>;
  static constexpr int CO = 16, TWO = 4;
  static constexpr int QS = TWO * X::PA * X::MA * CO;
  static constexpr int YW = TWO * X::ADV;
  static constexpr int YS = CO * X::ADV * YW;
  static constexpr size_t SMEM = (size_t)(QS + YS) * sizeof(float);
};

template <int MO, int RO, int MI, typename YT>
__global__ void __launch_bounds__(256) output_transform_kernel(const float* __restrict__ M, YT* __restrict__ y,
                                                               Geometry g, const float* __restrict__ slopes) {
  using X = Ax<MO, RO, MI>;
  using C = OutCfg<MO, RO, MI>;
  constexpr NestedAxis A = make_axis(MO, RO, MI);
  extern __shared__ __align__(16) float smem[];
  float* Qs = smem;
  float* Ys = smem + C::QS;
  const int tid = threadIdx.x;
  const int wgroups = (g.tiles_w + C::TWO - 1) / C::TWO;
  int b = blockIdx.x;
  const int wg = b % wgroups;
  b /= wgroups;
  const int ah = b % g.tiles_h;
  const int n = b / g.tiles_h;
  const int co0 = blockIdx.y * C::CO;
  const int aw0 = wg * C::TWO;

#pragma unroll
  for (int ph = 0; ph < X::NPH; ++ph) {
#pragma unroll
    for (int pw = 0; pw < X::NPH; ++pw) {
      __syncthreads();
      // pass A: along w, Q[tile][p_h][q_w][co]
      for (int task = tid; task < C::CO * C::TWO * X::PA; task += blockDim.x) {
        const int co = task % C::CO;
        const int tile = (task / C::CO) % C::TWO;
        const int p_h = task / (C::CO * C::TWO);
        const int aw = aw0 + tile;
        float mv[X::PA], qv[X::MA];
        if (aw < g.tiles_w) {
          const long long t = ((((long long)n * g.tiles_h + ah) * g.tiles_w + aw) * X::NPH + ph) * X::NPH + pw;
          const float* src = M + ((long long)(p_h * X::PA) * g.T_pad + t) * g.cout_pad + co0 + co;
          const long long step = (long long)g.T_pad * g.cout_pad;
#pragma unroll
          for (int p_w = 0; p_w < X::PA; ++p_w) mv[p_w] = __ldg(src + p_w * step);
        } else {
#pragma unroll
          for (int p_w = 0; p_w < X::PA; ++p_w) mv[p_w] = 0.f;
        }
        out_axis<MO, RO, MI>(mv, qv);
#pragma unroll
        for (int q = 0; q < X::MA; ++q) Qs[((tile * X::PA + p_h) * X::MA + q) * C::CO + co] = qv[q];
      }
      __syncthreads();
      // pass B: along h, scatter kept outputs into Ys[co][i][tile*adv + j]
      for (int task = tid; task < C::CO * C::TWO * X::MA; task += blockDim.x) {
        const int co = task % C::CO;
        const int tile = (task / C::CO) % C::TWO;
        const int q_w = task / (C::CO * C::TWO);
        if (!keep(A, pw, q_w)) continue;
        float mv[X::PA], yv[X::MA];
#pragma unroll
        for (int p_h = 0; p_h < X::PA; ++p_h) mv[p_h] = Qs[((tile * X::PA + p_h) * X::MA + q_w) * C::CO + co];
        out_axis<MO, RO, MI>(mv, yv);
        const int jw = tile * X::ADV + A.shift[pw] + out_pos(A, q_w);
#pragma unroll
        for (int q_h = 0; q_h < X::MA; ++q_h) {
          if (keep(A, ph, q_h)) {
            const int ih = A.shift[ph] + out_pos(A, q_h);
            Ys[(co * X::ADV + ih) * C::YW + jw] = yv[q_h];
          }
        }
      }
    }
  }
  __syncthreads();
  // cooperative store (rows of TWO*adv consecutive outputs)
  for (int idx = tid; idx < C::CO * X::ADV * C::YW; idx += blockDim.x) {
    const int j = idx % C::YW;
    const int i = (idx / C::YW) % X::ADV;
    const int co = idx / (C::YW * X::ADV);
    const int coe = co0 + co;
    if (coe >= g.cout_e) continue;
    const int gi = ah * X::ADV + i, gj = aw0 * X::ADV + j;
    if (gi >= g.Hq || gj >= g.Wq) continue;
    int c = coe, Y = gi, Xc = gj;
    if (g.mode == 2) {
      const int f = coe / g.Cout;
      c = coe % g.Cout;
      Y = 2 * gi + f / 2;
      Xc = 2 * gj + f % 2;
    }
    if (Y >= g.Ho || Xc >= g.Wo) continue;
    float v = Ys[idx];
    if (slopes) v = v >= 0.f ? v : slopes[c] * v;
    y[(((long long)n * g.Cout + c) * g.Ho + Y) * g.Wo + Xc] = from_f<YT>(v);
  }
}

}  // namespace nw

namespace nw {

template <int MO, int RO, int MI, typename YT>
static nw_status_t output_launch(const nw_plan_st* p, const Geometry& g, const float* M, void* y, cudaStream_t s) {
  using C = OutCfg<MO, RO, MI>;
  auto kern = output_transform_kernel<MO, RO, MI, YT>;
  static bool attr_done = false;
  if (!attr_done) {
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::SMEM) != cudaSuccess)
      return NW_ERR_CUDA;
    attr_done = true;
  }
  const int wgroups = (g.tiles_w + C::TWO - 1) / C::TWO;
  const long long gx = (long long)g.N * g.tiles_h * wgroups;
  dim3 grid((unsigned)gx, (unsigned)((g.cout_e + C::CO - 1) / C::CO));
  LaunchScope scope_("output_transform", s);
  kern<<<grid, 256, C::SMEM, s>>>(M, static_cast<YT*>(y), g, p->prelu ? p->slopes : nullptr);
  return check_launch();
}

template <int MO, int RO, int MI>
nw_status_t output_impl(const nw_plan_st* p, const Geometry& g, const float* M, void* y, cudaStream_t s) {
  if (p->dtype == NW_DTYPE_BF16) return output_launch<MO, RO, MI, __nv_bfloat16>(p, g, M, y, s);
  return output_launch<MO, RO, MI, float>(p, g, M, y, s);
}

}  // namespace nw
