// xform_523.cu -- input / output transform kernels for the mixed nested F(5,2) (x) F(3,3)
// (outer kernel over a 2-tile grid: filters of up to 6 taps per phase, R8).
#include "input_transform.cuh"
#include "output_transform.cuh"
#include "fused_small.cuh"

namespace nw {
template nw_status_t input_impl<5, 2, 3>(const nw_plan_st*, const Geometry&, const void*, void*, cudaStream_t);
template nw_status_t output_impl<5, 2, 3>(const nw_plan_st*, const Geometry&, const float*, void*, cudaStream_t);
template nw_status_t output_impl_pre<5, 2, 3>(const nw_plan_st*, const Geometry&, const float*, void*, cudaStream_t);
template nw_status_t output_impl_pre2<5, 2, 3>(const nw_plan_st*, const Geometry&, const float*, void*, cudaStream_t);
template nw_status_t fused_c1_impl<5, 2, 3>(const nw_plan_st*, const Geometry&, const void*, const void*, void*, void*,
                                                  cudaStream_t);
}  // namespace nw
