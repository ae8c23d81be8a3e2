// fgf_k_lowres_v3.cu -- the default K13 variant for fp32 samples (G 4, K 9/17, no sample ring,
// <= 160 threads x 3 CTAs/SM) in a translation unit of its own: its code generation through
// nvcc's split-compile path then does not depend on which other kernels share the unit
// (see the Makefile).
#include "fgf_lowres_launch.cuh"

namespace fgf {

int launch_lowres_v3_f32(const LowresParams& lp, const LrGeom& g, int images, const Plan& P,
                         cudaStream_t st) {
    return launch_lowres_gray_g<1, 4, 9, 17, false, 160, 3>(lp, g, images, P, st);
}

}  // namespace fgf
