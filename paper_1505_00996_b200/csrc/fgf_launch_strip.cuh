// fgf_launch_strip.cuh -- launchers of the strip engine (K1 statistics + coefficients, K3
// box of a, b), included by fgf_k_stats.cu and fgf_k_mean.cu, which instantiate one MODE each.
#pragma once
#include "fgf_host.cuh"

namespace fgf {

// measured (config 4): prefix sums win at r' = 32 (s = 1: 22.8 -> 15.6 ms per 32 images), lose at
// r' = 15, 16 (configs 2, 1 s=1, 4 s=2)
constexpr int kHpreR = 24;

template <int MODE, int CI, int CP, int NT, int G_ = 0>
int launch_strip_g(const StripParams& sp0, int images, const Plan& P, cudaStream_t st) {
    using C = StripConfig<MODE, CI, CP, NT, G_>;
    StripParams sp = sp0;
    sp.VP = NT + 2 * P.R + C::K + 1;
    const size_t smem = C::smem(sp.VP);
    if (smem > 227 * 1024) return FGF_ERR_UNSUPPORTED;
    // Segment height: ~4 waves of 148 SMs, a multiple of G rows, between 4G (and 2R) and 64
    // (256 for r' >= 16).
    const long long want = 4LL * 148;
    const long long strips_imgs = (long long)P.strips * images;
    long long th = (P.h * strips_imgs + want - 1) / want;
    th = std::max<long long>(th, std::max(4 * C::G, 2 * P.R));
    // wide windows (r' >= 16) amortise their 2r'+1 warm-up rows over taller segments: config 4
    // s = 1 15.38 -> 14.72 ms per 32 images, s = 2 35.09 -> 34.77 ms per 256 images; narrow
    // ones keep 64 (config 3's colour statistics are slower with taller segments)
    long long thmax = P.R >= 16 ? 256 : 64;
    if (const char* e = dev_env("FGF_STRIP_THMAX")) thmax = atoi(e);
    int TH = (int)std::min<long long>(thmax, th);
    // balanced segments: the same segment count with equal heights, no short last segment
    // (config 3: 64 + 64 + 64 + 64 + 14 -> 5 x 54 rows, 1.982 -> 1.961 ms)
    TH = (P.h + (P.h + TH - 1) / TH - 1) / ((P.h + TH - 1) / TH);
    TH = (TH + C::G - 1) / C::G * C::G;
    sp.TH = TH;
    sp.TW = P.TW;
    dim3 grid(P.strips, (P.h + TH - 1) / TH, images);
    // wide windows: prefix-sum horizontal phase (restart-free); measured threshold below
    int hpre_r = kHpreR;
    if (const char* e = dev_env("FGF_HPRE_R")) hpre_r = atoi(e);
    // (instantiated for gray 1/1 and colour 3/1, 3/3 -- the channel layouts BASELINE.json uses)
    constexpr bool HP_OK = (CI == 1 && CP == 1) || (CI == 3 && (CP == 1 || CP == 3));
    auto kern = box_strip_kernel<MODE, CI, CP, NT, G_, 0, false>;
    if constexpr (HP_OK) {
        if (P.R >= hpre_r) kern = box_strip_kernel<MODE, CI, CP, NT, G_, 0, true>;
    }
    set_smem(kern, smem);
    ProfScope ps(MODE == MODE_STATS ? KIND_STATS : KIND_MEAN, st);
    kern<<<grid, NT, smem, st>>>(sp);
    ++g_last_launches;
    return last_error();
}

// The default G assumes the worst-case padded row (r' up to the strip limit); colour
// statistics (13 / 21 fp64 maps) then get G = 1 or 2.  With r' <= 16 the real rows are short
// enough for more rows per batch (fewer barriers, longer runs).
template <int MODE, int CI, int CP, int NT>
int launch_strip_t(const StripParams& sp, int images, const Plan& P, cudaStream_t st) {
    constexpr bool MEANLIKE = MODE == MODE_MEAN;
    if (CI == 3 && NT == 256 && P.R <= 16 && dev_env("FGF_STRIP_WORSTG") == nullptr) {
        constexpr int GC = (MEANLIKE || CP == 1) ? 4 : 2;
        const int rc = launch_strip_g<MODE, CI, CP, NT, GC>(sp, images, P, st);
        if (rc != FGF_ERR_UNSUPPORTED) return rc;
    }
    // gray box of a, b at 12 <= r' < 24: 8 rows per batch (measured: config 4 s=2 K3 2.44 -> 2.27 ms
    // per 64 images; the statistics kernel was slower with 8)
    if (MEANLIKE && CI == 1 && CP == 1 && NT == 256 && P.R >= 12 && P.R < kHpreR &&
        dev_env("FGF_STRIP_WORSTG") == nullptr) {
        const int rc = launch_strip_g<MODE, CI, CP, NT, 8>(sp, images, P, st);
        if (rc != FGF_ERR_UNSUPPORTED) return rc;
    }
    return launch_strip_g<MODE, CI, CP, NT>(sp, images, P, st);
}

template <int MODE, int CI, int CP>
int launch_strip_nt(const StripParams& sp, int images, const Plan& P, cudaStream_t st) {
    if constexpr (MODE == MODE_STATS && CI == 3) {
        // colour statistics (21 / 13 fp64 running sums, ~230 registers): small CTAs, several
        // per SM instead of one of 256 threads -- 128 threads: 0.565 -> 0.493 ms (config 3),
        // 0.066 -> 0.060 ms (config 2); 64 threads where r' <= 8: 0.475 ms (config 3);
        // FGF_STATS_NT256=1 keeps the plan's width
        const bool keep = dev_env("FGF_STATS_NT256") != nullptr;
        if (!keep && 64 - 2 * P.R >= 48) {       // narrow windows: 64 threads (config 3 0.475 ms)
            Plan Q = P;
            Q.nt = 64;
            Q.TW = std::min(P.w, 64 - 2 * P.R);
            Q.strips = (P.w + Q.TW - 1) / Q.TW;
            return launch_strip_t<MODE, CI, CP, 64>(sp, images, Q, st);
        }
        if (!keep && 128 - 2 * P.R >= 64) {
            Plan Q = P;
            Q.nt = 128;
            Q.TW = std::min(P.w, 128 - 2 * P.R);
            Q.strips = (P.w + Q.TW - 1) / Q.TW;
            return launch_strip_t<MODE, CI, CP, 128>(sp, images, Q, st);
        }
    }
    if constexpr (MODE == MODE_MEAN && CI == 3 && CP == 1) {
        // colour box of a, b (4 maps per CTA; alone or as one of the C_p groups): 128-thread
        // CTAs -- config 3 K3 0.361 -> 0.337 ms, config 2 0.042 -> 0.033 ms;
        // FGF_MEAN_NT256=1 keeps the plan's width
        if (dev_env("FGF_MEAN_NT256") == nullptr && 128 - 2 * P.R >= 64) {
            Plan Q = P;
            Q.nt = 128;
            Q.TW = std::min(P.w, 128 - 2 * P.R);
            Q.strips = (P.w + Q.TW - 1) / Q.TW;
            return launch_strip_t<MODE, CI, CP, 128>(sp, images, Q, st);
        }
    }
    if (P.nt == 256) return launch_strip_t<MODE, CI, CP, 256>(sp, images, P, st);
    return launch_strip_t<MODE, CI, CP, 512>(sp, images, P, st);
}

template <int MODE>
int launch_strip(const StripParams& sp, int images, const Plan& P, cudaStream_t st) {
    if (MODE == MODE_MEAN && P.CI == 3 && P.CP > 1 && dev_env("FGF_MEAN_NOGROUP") == nullptr) {
        // colour box of a, b: the 4 C_p maps as C_p groups of 4 in one launch (the 3 / 1
        // kernel: 4 fp64 running sums per thread instead of 4 C_p, so 4 CTAs per SM instead of
        // one -- measured on config 3 below)
        StripParams g = sp;
        g.groups = P.CP;
        return launch_strip_nt<MODE, 3, 1>(g, images * P.CP, P, st);
    }
    switch (P.CI * 10 + P.CP) {
        case 11: return launch_strip_nt<MODE, 1, 1>(sp, images, P, st);
        case 12: return launch_strip_nt<MODE, 1, 2>(sp, images, P, st);
        case 13: return launch_strip_nt<MODE, 1, 3>(sp, images, P, st);
        case 14: return launch_strip_nt<MODE, 1, 4>(sp, images, P, st);
        case 31: return launch_strip_nt<MODE, 3, 1>(sp, images, P, st);
        case 32: return launch_strip_nt<MODE, 3, 2>(sp, images, P, st);
        case 33: return launch_strip_nt<MODE, 3, 3>(sp, images, P, st);
        case 34: return launch_strip_nt<MODE, 3, 4>(sp, images, P, st);
    }
    return FGF_ERR_SHAPE;
}

}  // namespace fgf
