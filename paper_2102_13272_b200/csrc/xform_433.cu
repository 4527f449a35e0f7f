// xform_433.cu -- input / output transform kernels for nested F(4,3) (x) F(3,3)
// (a larger outer tile: 12x12 outputs per slice, fewer transform points per output).
#include "input_transform.cuh"
#include "output_transform.cuh"
#include "fused_small.cuh"

namespace nw {
template nw_status_t input_impl<4, 3, 3>(const nw_plan_st*, const Geometry&, const void*, void*, cudaStream_t);
template nw_status_t output_impl<4, 3, 3>(const nw_plan_st*, const Geometry&, const float*, void*, cudaStream_t);
template nw_status_t output_impl_pre<4, 3, 3>(const nw_plan_st*, const Geometry&, const float*, void*, cudaStream_t);
template nw_status_t output_impl_pre2<4, 3, 3>(const nw_plan_st*, const Geometry&, const float*, void*, cudaStream_t);
template nw_status_t fused_c1_impl<4, 3, 3>(const nw_plan_st*, const Geometry&, const void*, const void*, void*, void*,
                                                  cudaStream_t);
}  // namespace nw
