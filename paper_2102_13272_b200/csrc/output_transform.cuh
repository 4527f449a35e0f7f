// output_transform.cuh -- G4: nested output transform fused with the store.
// Instantiated per axis combo in xform_*.cu.
//
// M layout [P][cout_pad][T_pad] (fp32): one warp owns 32 consecutive slices of one
// output channel, so every load of M is a 128-byte coalesced row.  Each thread
// keeps the 9x9 (M_a x M_a) output tile of its slice in registers: for each
// point row p_h it applies A^T_hat along w (factored, 25 -> 9) and accumulates
// A^T_hat[q_h][p_h] times that row into the tile (composite along h, zero
// coefficients skipped at compile time).  The tile then goes through a per-warp
// shared-memory stage so the stores walk whole output rows across the 32 slices
// (adjacent tiles are adjacent in w), applying the keep mask (redundant terms /
// coverage phases), the crop, the transposed-conv depth-to-space, PReLU and the
// dtype cast.
#pragma once
#include "transforms.cuh"

namespace nw {

struct AtHatF {
  float a[kMaxMa][kMaxPa];
};
template <int MO, int RO, int MI>
__host__ __device__ constexpr AtHatF make_athat() {
  AtHatF T{};
  NestedAxis A = make_axis(MO, RO, MI);
  for (int q = 0; q < A.Ma; ++q)
    for (int p = 0; p < A.Pa; ++p) T.a[q][p] = float(rdouble(at_hat(A, q, p)));
  return T;
}

template <int MO, int RO, int MI>
struct OutCfg {
  using X = Ax<MO, RO, MI>;
  static constexpr int WARPS = 8;
  static constexpr int STAGE = 32 * X::MA * X::MA + 1;  // floats per warp (odd stride per slice)
  static constexpr size_t SMEM = (size_t)WARPS * STAGE * sizeof(float);
};

template <int MO, int RO, int MI, typename YT>
__global__ void __launch_bounds__(256, 2) output_transform_kernel(const float* __restrict__ M, YT* __restrict__ y,
                                                                  Geometry g, const float* __restrict__ slopes) {
  using X = Ax<MO, RO, MI>;
  using C = OutCfg<MO, RO, MI>;
  constexpr NestedAxis A = make_axis(MO, RO, MI);
  constexpr AtHatF AT = make_athat<MO, RO, MI>();
  constexpr int MA = X::MA, PA = X::PA, NPH = X::NPH;
  extern __shared__ __align__(16) float smem[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  float* stage = smem + warp * C::STAGE;

  const long long t0 = (long long)blockIdx.x * 32;
  const int coe = blockIdx.y * C::WARPS + warp;
  if (coe >= g.cout_e) return;
  const long long t = t0 + lane;
  const bool valid = t < g.T;

  float Y[MA][MA];
#pragma unroll
  for (int i = 0; i < MA; ++i)
#pragma unroll
    for (int j = 0; j < MA; ++j) Y[i][j] = 0.f;

  const long long pstride = (long long)g.cout_pad * g.T_pad;   // between consecutive points
  const float* src = M + (long long)coe * g.T_pad + (valid ? t : 0);
#pragma unroll
  for (int p_h = 0; p_h < PA; ++p_h) {
    float mv[PA], qv[MA];
#pragma unroll
    for (int p_w = 0; p_w < PA; ++p_w) mv[p_w] = __ldg(src + (long long)(p_h * PA + p_w) * pstride);
    out_axis<MO, RO, MI>(mv, qv);
#pragma unroll
    for (int q_h = 0; q_h < MA; ++q_h) {
      if (AT.a[q_h][p_h] != 0.f) {
#pragma unroll
        for (int q_w = 0; q_w < MA; ++q_w) Y[q_h][q_w] = fmaf(AT.a[q_h][p_h], qv[q_w], Y[q_h][q_w]);
      }
    }
  }

  // stage the tile: stage[lane * MA*MA + q_h*MA + q_w]
#pragma unroll
  for (int q_h = 0; q_h < MA; ++q_h)
#pragma unroll
    for (int q_w = 0; q_w < MA; ++q_w) stage[lane * (MA * MA) + q_h * MA + q_w] = Y[q_h][q_w];
  __syncwarp();

  // store: index = (q_h, slice, q_w) so consecutive lanes walk one output row across slices
  int c = coe, fo_h = 0, fo_w = 0;
  if (g.mode == 2) {
    const int f = coe / g.Cout;
    c = coe % g.Cout;
    fo_h = f / 2;
    fo_w = f % 2;
  }
  const float slope = slopes ? slopes[c] : 0.f;
  const long long nslices = g.T - t0 < 32 ? g.T - t0 : 32;
  for (int idx = lane; idx < 32 * MA * MA; idx += 32) {
    const int q_w = idx % MA;
    const int s = (idx / MA) % 32;
    const int q_h = idx / (MA * 32);
    if (s >= nslices) continue;
    long long ts = t0 + s;
    const int phw = (int)(ts % NPH);
    ts /= NPH;
    const int phh = (int)(ts % NPH);
    ts /= NPH;
    const int aw = (int)(ts % g.tiles_w);
    ts /= g.tiles_w;
    const int ah = (int)(ts % g.tiles_h);
    const int n = (int)(ts / g.tiles_h);
    if (!keep(A, phh, q_h) || !keep(A, phw, q_w)) continue;
    const int gi = ah * X::ADV + A.shift[phh] + out_pos(A, q_h);
    const int gj = aw * X::ADV + A.shift[phw] + out_pos(A, q_w);
    if (gi >= g.Hq || gj >= g.Wq) continue;
    int Yr = gi, Xc = gj;
    if (g.mode == 2) {
      Yr = 2 * gi + fo_h;
      Xc = 2 * gj + fo_w;
      if (Yr >= g.Ho || Xc >= g.Wo) continue;
    }
    float v = stage[s * (MA * MA) + q_h * MA + q_w];
    if (slopes) v = v >= 0.f ? v : slope * v;
    y[(((long long)n * g.Cout + c) * g.Ho + Yr) * g.Wo + Xc] = from_f<YT>(v);
  }
}

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
  dim3 grid((unsigned)((g.T + 31) / 32), (unsigned)((g.cout_e + C::WARPS - 1) / C::WARPS));
  LaunchScope scope_("output_transform", s);
  kern<<<grid, 32 * C::WARPS, C::SMEM, s>>>(M, static_cast<YT*>(y), g, p->prelu ? p->slopes : nullptr);
  return check_launch();
}

template <int MO, int RO, int MI>
nw_status_t output_impl(const nw_plan_st* p, const Geometry& g, const float* M, void* y, cudaStream_t s) {
  if (p->dtype == NW_DTYPE_BF16) return output_launch<MO, RO, MI, __nv_bfloat16>(p, g, M, y, s);
  return output_launch<MO, RO, MI, float>(p, g, M, y, s);
}

}  // namespace nw
