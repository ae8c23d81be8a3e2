// fgf_k_mean.cu -- the strip engine's launches: K0, subsampling (Alg. 2 step 1, PAPER.md
// P:70-73), K1, box statistics + coefficients a, b (steps 2-4), and K3, box of a, b
// (step 5).
#include "fgf_launch_strip.cuh"

namespace fgf {

// K0: step 1 into compact fp32 low-res planes (s = 1 nearest: a conversion to fp32); planes
// [0, planes) from src, then planes2 more from src2 (I and p in one launch), into consecutive
// dst planes.
template <typename E>
int launch_subsample_e(const void* src, int planes, const void* src2, int planes2, float* dst,
                       const Plan& P, cudaStream_t st) {
    SubParams sp{src, dst, P.H, P.W, P.h, P.w, P.s, 8, src2 ? src2 : src, planes};
    dim3 grid((P.w + 255) / 256, (P.h + sp.rows_per_cta - 1) / sp.rows_per_cta, planes + planes2);
    ProfScope ps(KIND_SUB, st);
    const uintptr_t al = reinterpret_cast<uintptr_t>(src) |
                         (src2 ? reinterpret_cast<uintptr_t>(src2) : 0);
    const bool vec4 = P.s == 4 && (al & (4 * sizeof(E) - 1)) == 0 && (P.W % 4) == 0;
    if (P.sub == FGF_SUB_NEAREST)
        subsample_nearest_kernel<8, E><<<grid, 256, 0, st>>>(sp);
    else if (vec4)
        subsample_block_kernel<true, E><<<grid, 256, 0, st>>>(sp);
    else
        subsample_block_kernel<false, E><<<grid, 256, 0, st>>>(sp);
    ++g_last_launches;
    return last_error();
}

int launch_subsample2(const void* src, int planes, const void* src2, int planes2, float* dst,
                      const Plan& P, cudaStream_t st) {
    switch (P.dtype) {
        case FGF_F16: return launch_subsample_e<__half>(src, planes, src2, planes2, dst, P, st);
        case FGF_BF16: return launch_subsample_e<__nv_bfloat16>(src, planes, src2, planes2, dst, P, st);
        case FGF_U8: return launch_subsample_e<unsigned char>(src, planes, src2, planes2, dst, P, st);
    }
    return launch_subsample_e<float>(src, planes, src2, planes2, dst, P, st);
}

int launch_subsample(const void* src, float* dst, int planes, const Plan& P, cudaStream_t st) {
    return launch_subsample2(src, planes, nullptr, 0, dst, P, st);
}

template int launch_strip<MODE_STATS>(const StripParams&, int, const Plan&, cudaStream_t);
template int launch_strip<MODE_MEAN>(const StripParams&, int, const Plan&, cudaStream_t);

}  // namespace fgf
