// fgf_k_mean.cu -- K0: subsampling (Alg. 2 step 1) and K3: box of a, b
// (step 5).
#include "fgf_launch_strip.cuh"

namespace fgf {

// K0: step 1 into compact fp32 low-res planes (s = 1 nearest: a conversion to fp32).
template <typename E>
int launch_subsample_e(const void* src, float* dst, int planes, const Plan& P, cudaStream_t st) {
    SubParams sp{src, dst, P.H, P.W, P.h, P.w, P.s, 8};
    dim3 grid((P.w + 255) / 256, (P.h + sp.rows_per_cta - 1) / sp.rows_per_cta, planes);
    ProfScope ps(KIND_SUB, st);
    const bool vec4 = P.s == 4 && (reinterpret_cast<uintptr_t>(src) & (4 * sizeof(E) - 1)) == 0 &&
                      (P.W % 4) == 0;
    if (P.sub == FGF_SUB_NEAREST)
        subsample_nearest_kernel<8, E><<<grid, 256, 0, st>>>(sp);
    else if (vec4)
        subsample_block_kernel<true, E><<<grid, 256, 0, st>>>(sp);
    else
        subsample_block_kernel<false, E><<<grid, 256, 0, st>>>(sp);
    ++g_last_launches;
    return last_error();
}

int launch_subsample(const void* src, float* dst, int planes, const Plan& P, cudaStream_t st) {
    switch (P.dtype) {
        case FGF_F16: return launch_subsample_e<__half>(src, dst, planes, P, st);
        case FGF_BF16: return launch_subsample_e<__nv_bfloat16>(src, dst, planes, P, st);
        case FGF_U8: return launch_subsample_e<unsigned char>(src, dst, planes, P, st);
    }
    return launch_subsample_e<float>(src, dst, planes, P, st);
}

template int launch_strip<MODE_MEAN>(const StripParams&, int, const Plan&, cudaStream_t);

}  // namespace fgf
