// fgf_k_tiny.cu -- K6 (fgf_tiny.cuh): the single-kernel path for small gray images.
#include "fgf_host.cuh"
#include "fgf_tiny.cuh"

namespace fgf {

bool tiny_supports(const Plan& P) {
    return P.CI == 1 && P.CP == 1 && P.dtype == FGF_F32 && P.n <= (size_t)kTinyMaxN &&
           P.R <= kTinyMaxR && P.batch <= 64 && P.N <= (4u << 20);
}

int launch_tiny(const float* I, const float* p, float* q, const Plan& P, cudaStream_t st) {
    TinyParams tp{};
    tp.I = I; tp.p = p; tp.q = q;
    tp.H = P.H; tp.W = P.W; tp.h = P.h; tp.w = P.w; tp.s = P.s; tp.sub = P.sub; tp.R = P.R;
    tp.eps = P.eps; tp.k1 = P.k1; tp.k0 = P.k0;
    // output bands of ~4 rows per CTA (each CTA computes the low-res chain of the few rows its
    // band needs; measured on config 0: 4 / 8 / 16 / 32-row bands 10.8 / 11.4 / 15.9 / 20.5 us)
    int rows = 4;
    if (const char* e = dev_env("FGF_TINY_ROWS")) rows = std::max(1, atoi(e));   // development knob
    tp.bands = std::max(1, std::min(296, (P.H + rows - 1) / rows));
    const size_t smem = tiny_smem((int)P.n);
    set_smem(tiny_gray_kernel, smem);
    dim3 grid(tp.bands, P.batch);
    ProfScope ps(KIND_TINY, st);
    tiny_gray_kernel<<<grid, kTinyThreads, smem, st>>>(tp);
    ++g_last_launches;
    return last_error();
}

}  // namespace fgf
