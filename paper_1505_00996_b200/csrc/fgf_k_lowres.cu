// fgf_k_lowres.cu -- K13: the fused low-res chain for gray guidance (Alg. 2 steps 1-5 in one
// kernel, fgf_lowres.cuh): variant table, strip / segment geometry, launch.
#include "fgf_lowres_launch.cuh"

namespace fgf {

template <int CP>
int launch_lowres_gray_t(const LowresParams& lp0, int images, const Plan& P, cudaStream_t st,
                         bool dry) {
    // geometry from the whole call's batch, not the pipeline chunk's: every chunk of a call
    // then runs the same segments, so a chunked call equals the one-chunk call bit for bit
    LrGeom g;
    if (!lowres_geom<CP>(g, P.h, P.w, P.R, std::max(images, P.batch))) return FGF_ERR_UNSUPPORTED;
    if (dry) return FGF_OK;
    LowresParams lp = lp0;
    lp.TW = g.TW;
    lp.TH = g.TH;
    if (CP > 1) return launch_lowres_gray_g<CP, 4, 9, 9>(lp, g, images, P, st);
    if (P.dtype != FGF_F32) {   // reduced-precision inputs: the default variant and the wide one
        const bool h = P.dtype == FGF_F16;
        if (P.dtype == FGF_U8) {
            if (g.V == 3) return launch_lowres_v3<unsigned char>(lp, g, images, P, st);
            if (g.V == 0) return launch_lowres_gray_g<1, 4, 9, 9, true, 512, 1, unsigned char>(lp, g, images, P, st);
            return FGF_ERR_UNSUPPORTED;
        }
        if (g.V == 3)
            return h ? launch_lowres_v3<__half>(lp, g, images, P, st)
                     : launch_lowres_v3<__nv_bfloat16>(lp, g, images, P, st);
        if (g.V == 0)
            return h ? launch_lowres_gray_g<1, 4, 9, 9, true, 512, 1, __half>(lp, g, images, P, st)
                     : launch_lowres_gray_g<1, 4, 9, 9, true, 512, 1, __nv_bfloat16>(lp, g, images, P, st);
        return FGF_ERR_UNSUPPORTED;
    }
    switch (g.V) {
        case 0: return launch_lowres_gray_g<1, 4, 9, 9>(lp, g, images, P, st);
        case 1: return launch_lowres_gray_g<1, 8, 9, 9>(lp, g, images, P, st);
        case 2: return launch_lowres_gray_g<1, 4, 9, 9, false, 160, 4>(lp, g, images, P, st);
        case 3: return launch_lowres_v3<float>(lp, g, images, P, st);
    }
    return FGF_ERR_UNSUPPORTED;
}

// dry = true: only report whether K13 serves this plan (FGF_OK) or not.
int launch_lowres_gray(const LowresParams& lp, int images, const Plan& P, cudaStream_t st,
                       bool dry) {
    if (P.CI != 1) return FGF_ERR_UNSUPPORTED;
    // K13's horizontal restarts cost (2r' + 1) / K per output and its a, b ring 2r' + G + 1
    // rows: measured faster than the strip engine at r' = 4 and 8, slower at r' = 16 and 32
    // (config 4 at s = 8, 4, 2, 1), so wide windows take the strip engine.
    int rmax = 12;
    if (const char* e = dev_env("FGF_LR_RMAX")) rmax = atoi(e);
    if (P.R > rmax) return FGF_ERR_UNSUPPORTED;
    if (const char* e = dev_env("FGF_LOWRES")) {
        if (strcmp(e, "strip") == 0) return FGF_ERR_UNSUPPORTED;
    }
    if (P.dtype != FGF_F32 && P.CP != 1) return FGF_ERR_UNSUPPORTED;
    switch (P.CP) {
        case 1: {
            if (P.dtype != FGF_F32 && dry) {
                // only variants 3 and 0 exist for reduced-precision inputs
                LrGeom g;
                if (!lowres_geom<1>(g, P.h, P.w, P.R, std::max(images, P.batch))) return FGF_ERR_UNSUPPORTED;
                return (g.V == 3 || g.V == 0) ? FGF_OK : FGF_ERR_UNSUPPORTED;
            }
            return launch_lowres_gray_t<1>(lp, images, P, st, dry);
        }
        case 2: return launch_lowres_gray_t<2>(lp, images, P, st, dry);
    }
    return FGF_ERR_UNSUPPORTED;
}

}  // namespace fgf
