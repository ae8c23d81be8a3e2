// fgf_band.cuh -- row-band decomposition of ONE image across ranks (BASELINE.json config 4b,
// SURVEY §8(e)), host side, included by fgf_api.cu after the launch helpers.
//
// Rank k owns full-resolution rows [row0, row0 + rows) (row0 a multiple of s; the last band
// ends at H), i.e. low-res rows [y0, y1) = [row0/s, ceil((row0+rows)/s)) of the h = ceil(H/s)
// low-res rows.  Its rows upsample from low-res rows y0-1 .. y1 (R5); their mean_a, mean_b
// need a, b r' rows further and those need I', p' r' rows further again, so ONE exchange of
// HALO = 2r'+1 low-res rows of I' and p' with each neighbour makes everything after it local
// (the single-step variant of SURVEY §8(e)).  Windows clip at the global bounds because the
// extended band [e0, e1) = [y0 - HALO, y1 + HALO) is clipped to [0, h): at interior band
// edges the clipped windows only reach a, b rows this rank never uses.
//
//   subsample own rows into the extended planes -> exchange HALO rows with rank-1 / rank+1
//   (NCCL P2P in one group; or the one-process loop-back driver) -> low-res chain on the
//   extended band (K13 / strip engine, r' given) -> K4 on the own rows (global vertical map)
//
// Two-step mode (FGF_BAND_TWO_STEP, SURVEY §8(e)'s first form, BASELINE.json's "halo of
// ceil(r/s)+1 low-res rows"): exchange A sends r' rows of I', p'; the statistics and a, b of
// the OWN rows follow; exchange B sends r'+1 rows of a, b; the box of a, b then covers the
// own rows +-1 and K4 runs as above.  Two NCCL latencies instead of one, fewer bytes for
// colour guidance.
//
// The NCCL library is loaded at run time (dlopen "libnccl.so.2": the one torch already
// loaded when present), so libfgf.so itself has no link dependency on it.
#pragma once

#include <dlfcn.h>
#include <nccl.h>

namespace fgf {
namespace {

// ---------------------------------------------------------------- NCCL, loaded at run time
struct Nccl {
    bool tried = false, ok = false;
    decltype(&ncclGetUniqueId) getUniqueId = nullptr;
    decltype(&ncclCommInitRank) commInitRank = nullptr;
    decltype(&ncclCommDestroy) commDestroy = nullptr;
    decltype(&ncclSend) send = nullptr;
    decltype(&ncclRecv) recv = nullptr;
    decltype(&ncclGroupStart) groupStart = nullptr;
    decltype(&ncclGroupEnd) groupEnd = nullptr;
    decltype(&ncclCommGetAsyncError) commGetAsyncError = nullptr;   // optional
};
std::mutex g_nccl_mu;
Nccl g_nccl;

const Nccl* nccl() {
    std::lock_guard<std::mutex> lk(g_nccl_mu);
    if (!g_nccl.tried) {
        g_nccl.tried = true;
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (h) {
            g_nccl.getUniqueId = (decltype(g_nccl.getUniqueId))dlsym(h, "ncclGetUniqueId");
            g_nccl.commInitRank = (decltype(g_nccl.commInitRank))dlsym(h, "ncclCommInitRank");
            g_nccl.commDestroy = (decltype(g_nccl.commDestroy))dlsym(h, "ncclCommDestroy");
            g_nccl.send = (decltype(g_nccl.send))dlsym(h, "ncclSend");
            g_nccl.recv = (decltype(g_nccl.recv))dlsym(h, "ncclRecv");
            g_nccl.groupStart = (decltype(g_nccl.groupStart))dlsym(h, "ncclGroupStart");
            g_nccl.groupEnd = (decltype(g_nccl.groupEnd))dlsym(h, "ncclGroupEnd");
            g_nccl.commGetAsyncError =
                (decltype(g_nccl.commGetAsyncError))dlsym(h, "ncclCommGetAsyncError");
            g_nccl.ok = g_nccl.getUniqueId && g_nccl.commInitRank && g_nccl.commDestroy &&
                        g_nccl.send && g_nccl.recv && g_nccl.groupStart && g_nccl.groupEnd;
        }
    }
    return g_nccl.ok ? &g_nccl : nullptr;
}

// ---------------------------------------------------------------- band plan
struct BandPlan {
    int mode;                // FGF_BAND_SINGLE / FGF_BAND_TWO_STEP
    int H, W, h, w, s, sub, R, halo;
    int row0, rows;          // own full-res rows
    int y0, y1;              // own low-res rows
    int e0, e1;              // extended low-res rows of I', p' after (the first) exchange
    int f0, f1;              // two-step: rows of a, b after exchange B ([y0-r'-1, y1+r'+1))
    int CI, CP, NPL;         // planes exchanged: C_I (+ C_p unless self-guided)
    size_t ext_plane;        // floats per extended plane: (e1 - e0) * w
    size_t ab_plane;         // two-step: floats per a, b / mean plane: (f1 - f0) * w
    // workspace carve-up (bytes)
    size_t o_ext, o_lowres, o_mean, o_ab, o_abx, ws_total;
    Plan lp;                 // the low-res plan on the extended band (s = 1, radius r')
    Plan lpB;                // two-step: the plan of the box of a, b on rows [f0, f1)
};

int band_plan(BandPlan& B, int H, int W, int row0, int rows, int CI, int CP, int r, double eps,
              int s, int sub, int nranks, bool self_guided, int mode = FGF_BAND_SINGLE) {
    if (mode != FGF_BAND_SINGLE && mode != FGF_BAND_TWO_STEP) return FGF_ERR_PARAM;
    B.mode = mode;
    int rc = check_shape_params(1, H, W, CI, CP, r, eps, s, sub);
    if (rc) return rc;
    if (rows < 1 || row0 < 0 || row0 + rows > H) return FGF_ERR_SHAPE;
    if (row0 % s != 0 || ((row0 + rows) % s != 0 && row0 + rows != H)) return FGF_ERR_PARAM;
    B.H = H; B.W = W; B.s = s; B.sub = sub; B.CI = CI; B.CP = CP;
    B.h = lowres_dim(H, s);
    B.w = lowres_dim(W, s);
    B.R = radius_lowres(r, s);
    // single: 2r'+1 rows of I', p'; two-step: r' rows of I', p' (exchange A), then r'+1 rows
    // of a, b (exchange B)
    B.halo = mode == FGF_BAND_SINGLE ? 2 * B.R + 1 : B.R;
    B.row0 = row0; B.rows = rows;
    B.y0 = row0 / s;
    B.y1 = lowres_dim(row0 + rows, s);
    // every band (so every neighbour) must hold a whole halo, unless it is alone
    const int need = mode == FGF_BAND_SINGLE ? B.halo : B.R + 1;
    if (nranks > 1 && B.y1 - B.y0 < need) return FGF_ERR_PARAM;
    B.e0 = std::max(0, B.y0 - B.halo);
    B.e1 = std::min(B.h, B.y1 + B.halo);
    B.f0 = std::max(0, B.y0 - B.R - 1);
    B.f1 = std::min(B.h, B.y1 + B.R + 1);
    B.NPL = self_guided ? CI : CI + CP;
    B.ext_plane = (size_t)(B.e1 - B.e0) * B.w;
    B.ab_plane = (size_t)(B.f1 - B.f0) * B.w;
    if ((rc = make_plan(B.lp, 1, B.e1 - B.e0, B.w, CI, CP, B.R, eps, 1, FGF_SUB_NEAREST)))
        return rc;
    B.o_ext = 0;
    B.o_lowres = align_up(B.NPL * B.ext_plane * sizeof(float));
    if (mode == FGF_BAND_SINGLE) {
        B.o_mean = B.o_lowres + align_up(plan_ws(B.lp, false));
        B.ws_total = B.o_mean + align_up((size_t)B.lp.NC * B.ext_plane * sizeof(float));
        return FGF_OK;
    }
    if ((rc = make_plan(B.lpB, 1, B.f1 - B.f0, B.w, CI, CP, B.R, eps, 1, FGF_SUB_NEAREST)))
        return rc;
    const size_t nc = (size_t)B.lp.NC;
    B.o_abx = B.o_lowres;                                            // a, b of the ext rows
    B.o_ab = B.o_abx + align_up(nc * B.ext_plane * sizeof(float));    // a, b rows [f0, f1)
    B.o_mean = B.o_ab + align_up(nc * B.ab_plane * sizeof(float));    // mean rows [f0, f1)
    B.ws_total = B.o_mean + align_up(nc * B.ab_plane * sizeof(float));
    return FGF_OK;
}

// Two-step: statistics + a, b on the extended I', p' rows (strip engine K1), then the own
// rows copied into the a, b buffer at their place in [f0, f1).
int band_stats_ab(const BandPlan& B, char* ws, cudaStream_t st, bool self_guided) {
    const float* ext = reinterpret_cast<const float*>(ws + B.o_ext);
    float* abx = reinterpret_cast<float*>(ws + B.o_abx);
    float* ab = reinterpret_cast<float*>(ws + B.o_ab);
    const Plan& P = B.lp;
    StripParams sp{};
    sp.srcI = ext; sp.imgI = (long long)B.CI * P.n; sp.planeI = (int)P.n;
    sp.srcP = self_guided ? ext : ext + B.CI * B.ext_plane;
    sp.imgP = (long long)B.CP * P.n; sp.planeP = (int)P.n;
    sp.row = P.w; sp.col = 1;
    sp.h = P.h; sp.w = P.w; sp.R = P.R; sp.eps = P.eps;
    sp.k1 = 1.0f; sp.k0 = 0.0f;
    sp.dst = abx;
    int rc = launch_strip<MODE_STATS>(sp, 1, P, st);
    if (rc) return rc;
    const size_t row_bytes = (size_t)(B.y1 - B.y0) * B.w * sizeof(float);
    if (cudaMemcpy2DAsync(ab + (size_t)(B.y0 - B.f0) * B.w, B.ab_plane * sizeof(float),
                          abx + (size_t)(B.y0 - B.e0) * B.w, B.ext_plane * sizeof(float),
                          row_bytes, P.NC, cudaMemcpyDeviceToDevice, st))
        return FGF_ERR_CUDA;
    return FGF_OK;
}

// Subsample the own rows into the extended planes (rows [y0 - e0, y1 - e0) of each plane).
int band_prepare(const BandPlan& B, const float* I, const float* p, char* ws, cudaStream_t st) {
    float* ext = reinterpret_cast<float*>(ws + B.o_ext);
    Plan sp{};
    sp.H = B.rows; sp.W = B.W; sp.s = B.s; sp.sub = B.sub;   // the band's own mode (R3 / R4)
    sp.h = B.y1 - B.y0; sp.w = B.w;
    const size_t own = (size_t)B.rows * B.W;
    for (int j = 0; j < B.NPL; ++j) {
        const float* src = j < B.CI ? I + j * own : p + (j - B.CI) * own;
        float* dst = ext + j * B.ext_plane + (size_t)(B.y0 - B.e0) * B.w;
        int rc = launch_subsample(src, dst, 1, sp, st);
        if (rc) return rc;
    }
    return FGF_OK;
}

// Halo geometry of plane j: the rows this rank sends up / down and receives from up / down.
struct Halo {
    float *send_up, *send_down, *recv_up, *recv_down;
    size_t n_up, n_down;     // floats (0 when there is no neighbour on that side)
};
Halo band_halo(const BandPlan& B, char* ws, int j, int rank, int nranks) {
    float* ext = reinterpret_cast<float*>(ws + B.o_ext) + j * B.ext_plane;
    Halo hl{};
    const int own0 = B.y0 - B.e0, own1 = B.y1 - B.e0;
    if (rank > 0) {
        hl.n_up = (size_t)(B.y0 - B.e0) * B.w;                 // = halo rows (validated)
        hl.send_up = ext + (size_t)own0 * B.w;
        hl.recv_up = ext;
    }
    if (rank < nranks - 1) {
        hl.n_down = (size_t)(B.e1 - B.y1) * B.w;
        hl.send_down = ext + (size_t)own1 * B.w - hl.n_down;
        hl.recv_down = ext + (size_t)own1 * B.w;
    }
    return hl;
}

// Two-step exchange B geometry of a, b plane m: r'+1 own rows each way, into [f0, y0), [y1, f1).
Halo band_halo_ab(const BandPlan& B, char* ws, int m, int rank, int nranks) {
    float* ab = reinterpret_cast<float*>(ws + B.o_ab) + m * B.ab_plane;
    Halo hl{};
    const int own0 = B.y0 - B.f0, own1 = B.y1 - B.f0;
    if (rank > 0) {
        hl.n_up = (size_t)(B.y0 - B.f0) * B.w;
        hl.send_up = ab + (size_t)own0 * B.w;
        hl.recv_up = ab;
    }
    if (rank < nranks - 1) {
        hl.n_down = (size_t)(B.f1 - B.y1) * B.w;
        hl.send_down = ab + (size_t)own1 * B.w - hl.n_down;
        hl.recv_down = ab + (size_t)own1 * B.w;
    }
    return hl;
}

// Low-res chain on the extended band, then K4 on the own rows.
int band_finish(const BandPlan& B, const float* I, float* q, char* ws, cudaStream_t st,
                bool self_guided) {
    float* mean = reinterpret_cast<float*>(ws + B.o_mean);
    int m0, m1;
    if (B.mode == FGF_BAND_SINGLE) {
        const float* ext = reinterpret_cast<const float*>(ws + B.o_ext);
        const float* Is = ext;
        const float* ps = self_guided ? ext : ext + B.CI * B.ext_plane;
        int rc = run_coefficients(Is, ps, mean, B.lp, ws + B.o_lowres, B.o_mean - B.o_lowres, st);
        if (rc) return rc;
        m0 = B.e0; m1 = B.e1;
    } else {
        // box of a, b on rows [f0, f1) (strip engine K3): correct on the own rows +-1
        const Plan& P = B.lpB;
        StripParams mp{};
        mp.srcI = reinterpret_cast<const float*>(ws + B.o_ab);
        mp.imgI = (long long)P.NC * P.n; mp.planeI = (int)P.n;
        mp.srcP = nullptr;
        mp.row = P.w; mp.col = 1;
        mp.dst = mean;
        mp.h = P.h; mp.w = P.w; mp.R = P.R; mp.eps = P.eps;
        mp.k1 = 1.0f; mp.k0 = 0.0f;
        int rc = launch_strip<MODE_MEAN>(mp, 1, P, st);
        if (rc) return rc;
        m0 = B.f0; m1 = B.f1;
    }
    Plan P{};
    P.batch = 1; P.H = B.rows; P.W = B.W; P.CI = B.CI; P.CP = B.CP; P.NC = B.lp.NC;
    P.h = m1 - m0; P.w = B.w; P.N = (size_t)B.rows * B.W; P.n = (size_t)(m1 - m0) * B.w; P.TR = 32;
    const Band band{B.H, B.h, B.row0, m0, m1 - m0};
    return launch_output(I, mean, q, 1, P, st, &band);
}

}  // namespace
}  // namespace fgf
