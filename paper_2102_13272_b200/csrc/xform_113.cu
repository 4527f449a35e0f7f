// xform_113.cu -- input / output transform kernels for F(1,1) (x) F(3,3), i.e. the
// single-level F(3,3) of the OLA-Winograd comparison path (Eq. 2.3).
#include "input_transform.cuh"
#include "output_transform.cuh"
#include "fused_small.cuh"

namespace nw {
template nw_status_t input_impl<1, 1, 3>(const nw_plan_st*, const Geometry&, const void*, void*, cudaStream_t);
template nw_status_t output_impl<1, 1, 3>(const nw_plan_st*, const Geometry&, const float*, void*, cudaStream_t);
template nw_status_t output_impl_pre<1, 1, 3>(const nw_plan_st*, const Geometry&, const float*, void*, cudaStream_t);
template nw_status_t output_impl_pre2<1, 1, 3>(const nw_plan_st*, const Geometry&, const float*, void*, cudaStream_t);
template nw_status_t fused_c1_impl<1, 1, 3>(const nw_plan_st*, const Geometry&, const void*, const void*, void*, void*,
                                                  cudaStream_t);
}  // namespace nw
