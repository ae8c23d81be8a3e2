// fgf_k_wide.cu -- K5 (fgf_wide.cuh): geometry, persistent grid and launch of the
// radius-independent fused chain for gray guidance: the exact guided filter (Alg. 1,
// PAPER.md P:49-65) at s = 1, and the low-res chain (Alg. 2 steps 2-5) for wide r'.
#include "fgf_host.cuh"
#include "fgf_wide.cuh"

namespace fgf {

namespace {

template <int CP>
constexpr int wide_g() { return CP == 1 ? 4 : (CP == 2 ? 2 : 1); }

int sm_count() {
    static int n = 0;
    if (n == 0) {
        int dev = 0, v = 0;
        if (cudaGetDevice(&dev) == cudaSuccess &&
            cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) == cudaSuccess && v > 0)
            n = v;
        else {
            cudaGetLastError();
            return 148;   // B200 (no device: size queries only)
        }
    }
    return n;
}

}  // namespace

// Strip / segment geometry: minimise (waves of items over the persistent CTAs) x (work per
// item ~ threads x rows streamed), with NT = round32(TW + 4R) <= 672 threads.
bool wide_geom(WideGeom& g, int h, int w, int R, int CP, int images, bool outq) {
    if (R < 4 || CP < 1 || CP > 4) return false;      // ring of 2R + 1 >= G rows
    // persistent CTAs: the fused filter (s = 1) runs 8-row batches, one CTA per SM; the
    // mean-maps mode 4-row batches, two CTAs per SM (measured on configs 1 and 4)
    const int Gr = outq && CP == 1 ? 8 : (CP == 1 ? 4 : (CP == 2 ? 2 : 1));
    const int slots = sm_count() * (outq && CP == 1 ? 1 : kWideCtasPerSM);
    double best = 1e300;
    for (int TW = 32; TW + 4 * R <= kWideMaxCols; TW += 32) {
        const int tw = std::min(TW, w);
        const int NT = (tw + 4 * R + 31) / 32 * 32;
        const int strips = (w + tw - 1) / tw;
        // segment counts: 1, 2, ... while a segment keeps >= 2R rows
        for (int segs = 1; segs <= std::max(1, h / std::max(16, 2 * R)); ++segs) {
            const int TH = (h + segs - 1) / segs;
            const long long items = (long long)strips * segs * images;
            const long long waves = (items + slots - 1) / slots;
            const double per_item = (double)NT * (TH + 2 * R + Gr + R / 2.0);
            const double cost = (double)waves * per_item;
            if (cost < best * 0.999) {
                best = cost;
                g.TW = tw; g.NT = NT; g.strips = strips; g.segs = segs; g.TH = TH;
                g.items = (int)std::min<long long>(items, 1LL << 30);
            }
            if (items >= 64LL * slots) break;
        }
        if (TW >= w) break;
    }
    if (best >= 1e300) return false;
    // development knobs (FGF_DEV=1): force the strip width / segment count (tests cover several
    // strips and segments on small images)
    if (const char* e = dev_env("FGF_WIDE_TW")) {
        const int tw = std::min(std::max(1, atoi(e)), w);
        if (tw + 4 * R > kWideMaxCols) return false;
        g.TW = tw;
        g.NT = (tw + 4 * R + 31) / 32 * 32;
        g.strips = (w + tw - 1) / tw;
    }
    if (const char* e = dev_env("FGF_WIDE_SEGS")) {
        g.segs = std::min(std::max(1, atoi(e)), h);
        g.TH = (h + g.segs - 1) / g.segs;
        g.segs = (h + g.TH - 1) / g.TH;
    }
    g.items = (int)std::min<long long>((long long)g.strips * g.segs * images, 1LL << 30);
    g.grid = std::min(g.items, slots);
    if (const char* e = dev_env("FGF_WIDE_GRID")) g.grid = std::max(1, std::min(g.grid, atoi(e)));
    g.R = R;
    g.ring_bytes = align_up((size_t)g.grid * (2 * R + 1) * 2 * CP * g.TW * sizeof(float));
    return true;
}

// Ring bytes that cover every geometry wide_geom can return for radius R (any image count).
size_t wide_ring_reserve(int R, int CP) {
    const int twmax = kWideMaxCols - 4 * R;
    if (twmax < 32) return 0;
    return align_up((size_t)sm_count() * kWideCtasPerSM * (2 * R + 1) * 2 * CP * twmax *
                    sizeof(float));
}

// Contiguous, 16-byte-aligned fp32 sample rows: TMA bulk copies can stage them.
bool wide_bulk_ok(const WideParams& wp) {
    // development knob FGF_WIDE_BULK=1: TMA bulk staging (measured slower than the per-thread
    // cp.async staging: config 4 s = 1 13.85 vs 12.92 ms per 32 images, config 1 0.218 vs 0.205 ms)
    if (!dev_env("FGF_WIDE_BULK")) return false;
    const uintptr_t a = reinterpret_cast<uintptr_t>(wp.srcI) | reinterpret_cast<uintptr_t>(wp.srcP);
    return wp.col == 1 && (a & 15u) == 0 && wp.row % 4 == 0 && wp.imgI % 4 == 0 &&
           wp.imgP % 4 == 0 && wp.planeP % 4 == 0 && wp.w % 4 == 0;
}

template <int CP, bool OUTQ, typename E, int G = wide_g<CP>(), int MINB = kWideCtasPerSM,
          bool BULK = false>
int launch_wide_t(const WideParams& wp0, const WideGeom& g, cudaStream_t st) {
    auto kern = wide_gray_kernel<CP, G, OUTQ, E, MINB, BULK>;
    WideParams wp = wp0;
    wp.TW = g.TW; wp.TH = g.TH; wp.strips = g.strips; wp.segs = g.segs; wp.items = g.items;
    wp.L = WideCfg<CP, G, BULK ? 2 : (sizeof(E) == 4 ? 1 : 0)>::layout(g.TW, g.R);
    if (wp.L.total > 227 * 1024) return FGF_ERR_UNSUPPORTED;
    set_smem(kern, wp.L.total);
    // persistent grid: as many CTAs as fit on the GPU at once (at most the geometry's)
    int occ = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, g.NT, wp.L.total) != cudaSuccess ||
        occ < 1)
        return FGF_ERR_CUDA;
    const int grid = std::min(g.grid, sm_count() * std::min(occ, MINB));
    ProfScope ps(KIND_WIDE, st);
    kern<<<grid, g.NT, wp.L.total, st>>>(wp);
    ++g_last_launches;
    return last_error();
}

template <bool OUTQ>
int launch_wide_cp(const WideParams& wp, const WideGeom& g, int CP, int dtype, cudaStream_t st) {
    if (dtype != FGF_F32) {
        if (CP != 1) return FGF_ERR_UNSUPPORTED;
        switch (dtype) {
            case FGF_F16: return launch_wide_t<1, OUTQ, __half>(wp, g, st);
            case FGF_BF16: return launch_wide_t<1, OUTQ, __nv_bfloat16>(wp, g, st);
            case FGF_U8: return launch_wide_t<1, OUTQ, unsigned char>(wp, g, st);
        }
        return FGF_ERR_UNSUPPORTED;
    }
    // default: the fused filter (s = 1) in 8-row batches, one CTA per SM (152 registers);
    // the mean-maps mode in 4-row batches, two CTAs per SM (80 registers).  FGF_WIDE_V=0 / 1
    // (development knob) forces the 4-row / 8-row variant.
    int v = OUTQ ? 1 : 0;
    if (const char* e = dev_env("FGF_WIDE_V")) v = atoi(e);   // 0, 1; 2: 6-row batches, one CTA/SM
    const bool bulk = wide_bulk_ok(wp);
    switch (CP) {
        case 1:
            if (v == 2) return launch_wide_t<1, OUTQ, float, 6, 1>(wp, g, st);
            if (v == 1)
                return bulk ? launch_wide_t<1, OUTQ, float, 8, 1, true>(wp, g, st)
                            : launch_wide_t<1, OUTQ, float, 8, 1>(wp, g, st);
            return bulk ? launch_wide_t<1, OUTQ, float, 4, kWideCtasPerSM, true>(wp, g, st)
                        : launch_wide_t<1, OUTQ, float>(wp, g, st);
    }
    return FGF_ERR_UNSUPPORTED;
}

int launch_wide(const WideParams& wp, const WideGeom& g, int CP, int dtype, bool outq,
                cudaStream_t st) {
    return outq ? launch_wide_cp<true>(wp, g, CP, dtype, st)
                : launch_wide_cp<false>(wp, g, CP, dtype, st);
}

bool wide_supports(int CP, int dtype) { return CP == 1 && dtype >= FGF_F32 && dtype <= FGF_U8; }

}  // namespace fgf
