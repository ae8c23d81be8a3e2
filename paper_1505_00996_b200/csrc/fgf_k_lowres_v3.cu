// fgf_k_lowres_v3.cu -- the default K13 variant (G 4, K 9/17, no sample ring, <= 160 threads x
// 3 CTAs/SM) for ONE sample type, FGF_V3_ELEM (float, __half, __nv_bfloat16, uint8_t).
// The Makefile compiles this file once per sample type into a unit of its own, each through
// tools/nvcc_pick.py, which keeps the split-compile outcome with the kernel's indices on the
// uniform datapath (nvcc's split-compile output varies from run to run, build).
#include "fgf_lowres_launch.cuh"

#ifndef FGF_V3_ELEM
#define FGF_V3_ELEM float
#endif

namespace fgf {

template <typename E>
int launch_lowres_v3(const LowresParams& lp, const LrGeom& g, int images, const Plan& P,
                     cudaStream_t st) {
    return launch_lowres_gray_g<1, 4, 9, 17, false, 160, 3, E>(lp, g, images, P, st);
}
template int launch_lowres_v3<FGF_V3_ELEM>(const LowresParams&, const LrGeom&, int, const Plan&,
                                           cudaStream_t);

}  // namespace fgf
