// dispatch.cu -- route a geometry's axis kernel (m_o, r_o, m_i) to its compiled transform kernels
// (the plan's nested kernel, or F(1,1) (x) F(3,3) = single-level F(3,3) for the OLA path).
#include <cstdlib>

#include "nw_internal.h"

namespace nw {

template <int MO, int RO, int MI>
nw_status_t input_impl(const nw_plan_st*, const Geometry&, const void*, void*, cudaStream_t);
template <int MO, int RO, int MI>
nw_status_t output_impl(const nw_plan_st*, const Geometry&, const float*, void*, cudaStream_t);
template <int MO, int RO, int MI>
nw_status_t output_impl_pre(const nw_plan_st*, const Geometry&, const float*, void*, cudaStream_t);
template <int MO, int RO, int MI>
nw_status_t output_impl_pre2(const nw_plan_st*, const Geometry&, const float*, void*, cudaStream_t);

template <int MO, int RO, int MI>
nw_status_t fused_c1_impl(const nw_plan_st*, const Geometry&, const void*, const void*, void*, void*, cudaStream_t);
template <int MO, int RO, int MI>
nw_status_t fused_co_impl(const nw_plan_st*, const Geometry&, const void*, const void*, void*, void*, cudaStream_t);

#define NW_DISPATCH_AXIS(p, FN, ...)                                       \
  do {                                                                     \
    const int mo_ = g.mo, ro_ = g.ro, mi_ = g.mi;                          \
    if (mo_ == 3 && ro_ == 3 && mi_ == 3) return FN<3, 3, 3>(__VA_ARGS__); \
    if (mo_ == 2 && ro_ == 3 && mi_ == 2) return FN<2, 3, 2>(__VA_ARGS__); \
    if (mo_ == 3 && ro_ == 2 && mi_ == 3) return FN<3, 2, 3>(__VA_ARGS__); \
    if (mo_ == 2 && ro_ == 3 && mi_ == 3) return FN<2, 3, 3>(__VA_ARGS__); \
    if (mo_ == 1 && ro_ == 1 && mi_ == 3) return FN<1, 1, 3>(__VA_ARGS__); \
    if (mo_ == 4 && ro_ == 3 && mi_ == 3) return FN<4, 3, 3>(__VA_ARGS__); \
    if (mo_ == 5 && ro_ == 3 && mi_ == 3) return FN<5, 3, 3>(__VA_ARGS__); \
    if (mo_ == 4 && ro_ == 2 && mi_ == 3) return FN<4, 2, 3>(__VA_ARGS__); \
    if (mo_ == 5 && ro_ == 2 && mi_ == 3) return FN<5, 2, 3>(__VA_ARGS__); \
    return NW_ERR_UNSUPPORTED;                                             \
  } while (0)

nw_status_t launch_input_transform(const nw_plan_st* p, const Geometry& g, const void* x, void* V, cudaStream_t s) {
  NW_DISPATCH_AXIS(p, input_impl, p, g, x, V, s);
}

nw_status_t launch_output_transform(const nw_plan_st* p, const Geometry& g, const float* M, void* y, cudaStream_t s) {
  NW_DISPATCH_AXIS(p, output_impl, p, g, M, y, s);
}

nw_status_t launch_output_transform_pre(const nw_plan_st* p, const Geometry& g, const float* M, void* y,
                                        cudaStream_t s) {
  NW_DISPATCH_AXIS(p, output_impl_pre, p, g, M, y, s);
}

nw_status_t launch_output_transform_pre2(const nw_plan_st* p, const Geometry& g, const float* M, void* y,
                                         cudaStream_t s) {
  NW_DISPATCH_AXIS(p, output_impl_pre2, p, g, M, y, s);
}

bool fused_c1_eligible(const nw_plan_st* p, const Geometry& g) {
  static const int on = [] {
    const char* v = getenv("NW_FUSED_C1");
    return v ? atoi(v) : 1;
  }();
  return on && !p->depthwise && g.path == kPathNested && g.mode == 0 && g.cin_e == 1 && g.mi == 3 && g.nph == 1 && g.mo >= 2 &&
         g.Pa <= 30;  // V of 32 slices in shared memory: up to F(4,3) / F(5,2) (x) F(3,3)
}

// fp32 U per channel group, [group][CO][P_a][P_a rounded up to even]: at most 16 channels of
// padding and one float of row padding
size_t fused_c1_ws_bytes(const nw_plan_st* p, const Geometry& g) {
  (void)p;
  return (size_t)((g.cout_e + 15) / 16 * 16) * g.Pa * (g.Pa + 1) * 4;
}

nw_status_t launch_fused_c1(const nw_plan_st* p, const Geometry& g, const void* x, const void* U, void* y,
                            void* ws, size_t ws_bytes, cudaStream_t s) {
  NW_DISPATCH_AXIS(p, fused_c1_impl, p, g, x, U, y, ws_bytes >= fused_c1_ws_bytes(p, g) ? ws : nullptr, s);
}

// Single-kernel path for at most four contraction outputs (fused_smallout.cuh): C5's 9x9
// stride-2 deconvolution (Cout_e = 4 output phases), Table I's SRCNN 5x5 1 <- 32.
bool fused_co_eligible(const nw_plan_st* p, const Geometry& g) {
  static const int on = [] {
    const char* v = getenv("NW_FUSED_CO");
    return v ? atoi(v) : 1;
  }();
  const long long row_bytes = (long long)g.W * (p->dtype == NW_DTYPE_BF16 ? 2 : 4);
  return on && !p->depthwise && !p->prelu && p->math != NW_MATH_BF16 && g.path == kPathNested && g.SR == 1 &&
         g.nph == 1 && g.mi == 3 && g.cin_e >= 2 && g.cout_e <= 4 && (g.Pa == 25 || g.Pa == 30) &&
         row_bytes % 16 == 0;  // x windows arrive by TMA
}

nw_status_t launch_fused_co(const nw_plan_st* p, const Geometry& g, const void* x, const void* U, void* y, void* ws,
                            cudaStream_t s) {
  NW_DISPATCH_AXIS(p, fused_co_impl, p, g, x, U, y, ws, s);
}

}  // namespace nw
