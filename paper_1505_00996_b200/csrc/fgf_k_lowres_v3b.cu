// fgf_k_lowres_v3b.cu -- the default K13 variant (G 4, K 9/17, no sample ring, <= 160 threads x 3 CTAs/SM)
// for 8-bit samples, in a translation unit of its own: built through tools/nvcc_pick.py,
// which keeps the split-compile outcome with the kernel's indices on the uniform datapath
// (see the Makefile).
#include "fgf_lowres_launch.cuh"

namespace fgf {

template <typename E>
int launch_lowres_v3(const LowresParams& lp, const LrGeom& g, int images, const Plan& P,
                     cudaStream_t st) {
    return launch_lowres_gray_g<1, 4, 9, 17, false, 160, 3, E>(lp, g, images, P, st);
}
template int launch_lowres_v3<unsigned char>(const LowresParams&, const LrGeom&, int, const Plan&, cudaStream_t);

}  // namespace fgf
