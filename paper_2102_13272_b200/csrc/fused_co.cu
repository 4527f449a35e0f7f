// fused_co.cu -- instantiations of the single-kernel path for layers with Cout_e <= 4
// (fused_smallout.cuh) for every axis combo the dispatcher knows; combos whose P_a is not
// 25 or 30 return NW_ERR_UNSUPPORTED (the three-kernel path runs instead).
#include "fused_smallout.cuh"

namespace nw {
#define NW_FCO(MO, RO, MI)                                                                                      \
  template nw_status_t fused_co_impl<MO, RO, MI>(const nw_plan_st*, const Geometry&, const void*, const void*, \
                                                 void*, void*, cudaStream_t);
NW_FCO(3, 3, 3)
NW_FCO(2, 3, 2)
NW_FCO(3, 2, 3)
NW_FCO(2, 3, 3)
NW_FCO(1, 1, 3)
NW_FCO(4, 3, 3)
NW_FCO(5, 3, 3)
NW_FCO(4, 2, 3)
NW_FCO(5, 2, 3)
#undef NW_FCO
}  // namespace nw
