// fgf_lowres_launch.cuh -- K13 launch helpers shared by fgf_k_lowres.cu (geometry, dispatch,
// the other variants) and fgf_k_lowres_v3.cu (the default fp32 variant in a unit of its own).
#pragma once
#include "fgf_host.cuh"

namespace fgf {

// ---- K13: fused low-res chain (gray guidance), fgf_lowres.cuh
constexpr size_t kLrSmemMax = 227 * 1024;

// Kernel variants (rows per batch G, horizontal run lengths KA / KB); the first that fits
// is used unless FGF_LR_V selects one (development sweep).
//   0: G 4, K 9/9, sample ring        1: G 8, K 9/9, sample ring
//   2: G 4, K 9/9, no ring, <=160 threads x 4 CTAs/SM
//   3: G 4, K 9/17 (stage-B runs of 17), no ring, <= 3 CTAs/SM -- the default
// (measured on config 4, profiles/round1/k13_variants.txt: G 8 / K 17 and G 6 / K 13 without
// the ring, and a lane-pair split of the runs, were slower; so were K 5/17, K 7/17, K 7/9 and
// K 9/25; K 9/17 beat K 9/9 by 1.5 %)
constexpr int kLrNumVariants = 4;

// Strip geometry of K13: NT = round32(TW + 4R) <= 512 threads per CTA.
struct LrGeom {
    int NT = 0, TW = 0, strips = 0, TH = 0, V = -1;
    size_t smem = 0;
};

template <int CP, int G, int KA, int KB, bool RING = true, int MAXT = 512>
inline bool lowres_fits(LrGeom& g, int R, int v) {
    using C = LowresCfg<CP, G, KA, KB, RING>;
    const auto L = C::layout(g.NT, g.TW, g.TH, R);
    // both horizontal phases run concurrently on disjoint threads
    if (L.total > kLrSmemMax || G * (L.nrA + L.nrB) > g.NT || g.NT > MAXT) return false;
    g.smem = L.total;
    g.V = v;
    return true;
}

template <int CP>
inline bool lowres_fits_v(LrGeom& g, int R, int v) {
    if (CP > 1 && v != 0) return false;          // one variant for several p channels
    switch (v) {
        case 0: return lowres_fits<CP, 4, 9, 9>(g, R, v);
        case 1: return lowres_fits<CP, 8, 9, 9>(g, R, v);
        case 2: return lowres_fits<CP, 4, 9, 9, false, 160>(g, R, v);
        case 3: return lowres_fits<CP, 4, 9, 17, false, 160>(g, R, v);
    }
    return false;
}

template <int CP>
inline bool lowres_geom(LrGeom& g, int h, int w, int R, int images) {
    // Target ~160 threads (5 warps) per CTA: three CTAs per SM, halo overhead (TW + 4R) / TW.
    int want_nt = 160;
    if (const char* e = dev_env("FGF_LR_NT")) want_nt = atoi(e);
    LrGeom best;
    for (int ns = 1; ns <= w; ++ns) {
        const int TW = (w + ns - 1) / ns;
        if ((ns - 1) * TW >= w) continue;
        const int NT = (TW + 4 * R + 31) / 32 * 32;
        if (NT > 512) continue;
        const long long tot = (long long)ns * NT, btot = (long long)best.strips * best.NT;
        // closest to the target size; on ties the fewer total threads
        const bool better = best.NT == 0 || std::abs(NT - want_nt) < std::abs(best.NT - want_nt) ||
                            (std::abs(NT - want_nt) == std::abs(best.NT - want_nt) && tot < btot);
        if (better) { best.NT = NT; best.TW = TW; best.strips = ns; }
        if (NT < 64) break;
    }
    if (best.NT == 0) return false;
    // 4-column multiples when the rows allow it: 16-byte aligned strips for the bulk stores
    if (w % 4 == 0 && best.TW % 4 != 0) {
        const int TW4 = (best.TW + 3) & ~3;
        if ((TW4 + 4 * R + 31) / 32 * 32 == best.NT) {
            best.TW = TW4;
            best.strips = (w + TW4 - 1) / TW4;
        }
    }
    // Segment height: long segments amortise the 2r'+1 warm-up rows (up to h / 2 rows); small
    // batches (single images) get shorter segments so that ~2 waves of 3 CTAs per SM exist.
    const long long cols = (long long)best.strips * images;
    long long th = ((long long)h * cols + 2 * 3 * 148 - 1) / (2 * 3 * 148);
    // (cap: half the image height, at least 256 and at most 512 rows -- config 4 s = 4:
    // 512-row segments 3.90 -> 3.78 ms; s = 8: 256 (= h / 2) best; whole-image segments were
    // slower.  The upper bound keeps stage B's fp32 running column sums (R17) to <= 512
    // add / remove steps per segment, whatever the image height: ADVICE r1; an fp64 or
    // periodically re-summed variant measured 3-6 % slower on config 4)
    const long long cap = std::max<long long>(256, std::min<long long>(512, (h + 1) / 2));
    const long long thmin = std::max(8, 2 * R + 2);
    th = std::min<long long>(cap, std::max<long long>(th, thmin));
    // Small batches (fewer strip columns than CTA slots, 3 per SM): the segment count that
    // minimises waves x rows streamed per CTA (TH + ~4r' + 3 warm-up rows) -- a launch just
    // over a whole number of waves pays a nearly empty one (one 16384^2 image, 32 strips:
    // TH 296 = 448 CTAs 0.734 ms, TH 342 = 384 CTAs 0.652 ms, the ~2-wave rule's 148 0.682 ms)
    constexpr long long kSlots = 3LL * 148;
    if (cols < kSlots) {
        double best_cost = 1e300;
        for (long long segs = 1; segs <= h; ++segs) {
            const long long T = (h + segs - 1) / segs;
            if (T < thmin) break;
            if (T > cap) continue;
            const long long items = cols * ((h + T - 1) / T);
            const double cost = (double)((items + kSlots - 1) / kSlots) * (double)(T + 4 * R + 3);
            if (cost < best_cost * 0.999) { best_cost = cost; th = T; }
        }
    }
    if (const char* e = dev_env("FGF_LR_TH")) th = atoi(e);
    best.TH = (int)std::max<long long>(1, std::min<long long>(th, h));
    if (const char* e = dev_env("FGF_LR_V")) {
        if (lowres_fits_v<CP>(best, R, atoi(e))) { g = best; return true; }
        return false;
    }
    static const int order[kLrNumVariants] = {3, 0, 1, 2};   // measured: 3 fastest (config 4)
    for (int v : order)
        if (lowres_fits_v<CP>(best, R, v)) { g = best; return true; }
    return false;
}

template <int CP, int G, int KA, int KB, bool RING = true, int MAXT = 512, int MINB = 1,
          typename E = float>
int launch_lowres_gray_g(const LowresParams& lp, const LrGeom& g, int images, const Plan& P,
                         cudaStream_t st) {
    auto kern = lowres_gray_kernel<CP, G, KA, KB, RING, MAXT, MINB, E>;
    LowresParams lpl = lp;
    lpl.L = LowresCfg<CP, G, KA, KB, RING>::layout(g.NT, lp.TW, lp.TH, P.R);
    // TMA bulk stores of the staged output rows: every row segment and Os row 16-byte aligned
    lpl.bulk_out = P.w % 4 == 0 && lp.TW % 4 == 0 && lpl.L.PB % 4 == 0 && lpl.L.ROS % 4 == 0 &&
                   (reinterpret_cast<uintptr_t>(lp.dst) & 15u) == 0 &&
                   dev_env("FGF_LR_NOBULK") == nullptr;
    size_t smem = g.smem;
    // optional floor on the dynamic smem: caps K13 CTAs per SM so that the output pass of the
    // previous chunk can be co-resident (overlap experiment knob)
    if (const char* e = dev_env("FGF_LR_SMEM_MIN")) smem = std::max<size_t>(smem, (size_t)atoi(e));
    set_smem(kern, smem);
    dim3 grid(g.strips, (P.h + g.TH - 1) / g.TH, images);
    ProfScope ps(KIND_LOWRES, st);
    kern<<<grid, g.NT, smem, st>>>(lpl);
    ++g_last_launches;
    return last_error();
}

// The default variant (G 4, K 9/17, no sample ring, <= 160 threads x 3 CTAs/SM) for samples of
// type E; each element type is instantiated in a translation unit of its own
// (fgf_k_lowres_v3.cu compiled once per type, through tools/nvcc_pick.py).
template <typename E>
int launch_lowres_v3(const LowresParams& lp, const LrGeom& g, int images, const Plan& P,
                     cudaStream_t st);
extern template int launch_lowres_v3<float>(const LowresParams&, const LrGeom&, int, const Plan&, cudaStream_t);
extern template int launch_lowres_v3<__half>(const LowresParams&, const LrGeom&, int, const Plan&, cudaStream_t);
extern template int launch_lowres_v3<__nv_bfloat16>(const LowresParams&, const LrGeom&, int, const Plan&, cudaStream_t);
extern template int launch_lowres_v3<unsigned char>(const LowresParams&, const LrGeom&, int, const Plan&, cudaStream_t);

}  // namespace fgf
