// fgf_k_stats.cu -- K1: box statistics + coefficients a, b (Alg. 2 steps 2-4).
#include "fgf_launch_strip.cuh"

namespace fgf {
template int launch_strip<MODE_STATS>(const StripParams&, int, const Plan&, cudaStream_t);
}  // namespace fgf
