// fgf_band.cuh -- row-band decomposition of ONE image across ranks (BASELINE.json config 4b,
// SURVEY §8(e)), host side, included by fgf_api.cu after the launch helpers.
//
// Rank k owns full-resolution rows [row0, row0 + rows) (row0 a multiple of s; the last band
// ends at H), i.e. low-res rows [y0, y1) = [row0/s, ceil((row0+rows)/s)) of the h = ceil(H/s)
// low-res rows.  Its rows upsample from low-res rows y0-1 .. y1 (R5) -- or y1 + 1 when H is not
// a multiple of s: the map scale h / H then exceeds 1 / s, and the last rows of a band reach
// up to one row further (below y1 + 1/2, so the row after y1 is the last one: x = 1 extra row,
// 0 when h s = H); their mean_a, mean_b need a, b r' rows further and those need I', p' r' rows
// further again, so ONE exchange of HALO = 2r'+1+x low-res rows of I' and p' with each
// neighbour makes everything after it local (the single-step variant of SURVEY §8(e)).  Windows clip at the global bounds because the
// extended band [e0, e1) = [y0 - HALO, y1 + HALO) is clipped to [0, h): at interior band
// edges the clipped windows only reach a, b rows this rank never uses.
//
//   subsample own rows into the extended planes -> exchange HALO rows with rank-1 / rank+1
//   (NCCL P2P in one group; or the one-process loop-back driver) -> low-res chain on the
//   extended band (K13 / strip engine, r' given) -> K4 on the own rows (global vertical map)
//
// Two-step mode (FGF_BAND_TWO_STEP, SURVEY §8(e)'s first form, BASELINE.json's "halo of
// ceil(r/s)+1 low-res rows"): exchange A sends r' rows of I', p'; the statistics and a, b of
// the OWN rows follow; exchange B sends r'+1+x rows of a, b; the box of a, b then covers the
// own rows -1 .. +1+x and K4 runs as above.  Two NCCL latencies instead of one, fewer bytes for
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
        // FGF_NCCL_LIB (a development knob, honoured only with FGF_DEV=1): another library
        // with NCCL's point-to-point ABI -- tests/nccl_shim.cpp, which runs the multi-rank
        // band path as several processes on one GPU
        const char* lib = dev_env("FGF_NCCL_LIB");
        void* h = dlopen(lib && *lib ? lib : "libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
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
    int x;                   // 1 when h s != H: the own rows upsample from up to row y1 + 1
    int row0, rows;          // own full-res rows
    int y0, y1;              // own low-res rows
    int e0, e1;              // extended low-res rows of I', p' after (the first) exchange
    int f0, f1;              // two-step: rows of a, b after exchange B ([y0-r'-1-x, y1+r'+1+x))
    int CI, CP, NPL;         // planes exchanged: C_I (+ C_p unless self-guided)
    int r_full;              // r (full resolution)
    size_t ext_plane;        // floats per extended plane: (e1 - e0) * w
    size_t ab_plane;         // two-step: floats per a, b / mean plane: (f1 - f0) * w
    // workspace carve-up (bytes)
    size_t o_ext, o_lowres, o_mean, o_ab, o_abx, ws_total;
    Plan lp;                 // the low-res plan on the extended band (s = 1, radius r')
    Plan lpB;                // two-step: the plan of the box of a, b on rows [f0, f1)
    // overlapped single exchange (band_plan_overlap): the interior is the band's own image
    bool ovl = false;
    Plan pb;                 // the band's rows as an image (full resolution, s, r)
    int m0, m1;              // rows of the assembled mean maps: [y0 - 1, y1 + 1 + x) clipped
    int t0, t1, b0, b1;      // top / bottom edge strips of low-res rows (halo + 4r' own rows)
    Plan pe_t, pe_b;         // s = 1 plans of the edge strips (radius r')
    size_t o_slot, o_int, o_et, o_etw, o_etm, o_eb, o_ebw, o_ebm, o_fin;
};

// Halo geometry of plane j: the rows this rank sends up / down and receives from up / down.
struct Halo {
    float *send_up, *send_down, *recv_up, *recv_down;
    size_t n_up, n_down;     // floats (0 when there is no neighbour on that side)
};

int band_plan_overlap(BandPlan& B, bool self_guided, double eps);

int band_plan(BandPlan& B, int H, int W, int row0, int rows, int CI, int CP, int r, double eps,
              int s, int sub, int nranks, bool self_guided, int mode = FGF_BAND_SINGLE) {
    if (mode != FGF_BAND_SINGLE && mode != FGF_BAND_TWO_STEP) return FGF_ERR_PARAM;
    B.mode = mode;
    int rc = check_shape_params(1, H, W, CI, CP, r, eps, s, sub);
    if (rc) return rc;
    if (rows < 1 || row0 < 0 || row0 + rows > H) return FGF_ERR_SHAPE;
    if (row0 % s != 0 || ((row0 + rows) % s != 0 && row0 + rows != H)) return FGF_ERR_PARAM;
    B.H = H; B.W = W; B.s = s; B.sub = sub; B.CI = CI; B.CP = CP; B.r_full = r;
    B.h = lowres_dim(H, s);
    B.w = lowres_dim(W, s);
    B.R = radius_lowres(r, s);
    // single: 2r'+1+x rows of I', p'; two-step: r' rows of I', p' (exchange A), then r'+1+x
    // rows of a, b (exchange B).  Both directions exchange the same depth (one extra row above
    // when x = 1, unused), so every halo message has one size on both sides.
    B.x = (long long)B.h * s != H ? 1 : 0;
    B.halo = mode == FGF_BAND_SINGLE ? 2 * B.R + 1 + B.x : B.R;
    B.row0 = row0; B.rows = rows;
    B.y0 = row0 / s;
    B.y1 = lowres_dim(row0 + rows, s);
    // every band (so every neighbour) must hold a whole halo, unless it is alone
    const int need = mode == FGF_BAND_SINGLE ? B.halo : B.R + 1 + B.x;
    if (nranks > 1 && B.y1 - B.y0 < need) return FGF_ERR_PARAM;
    B.e0 = std::max(0, B.y0 - B.halo);
    B.e1 = std::min(B.h, B.y1 + B.halo);
    B.f0 = std::max(0, B.y0 - B.R - 1 - B.x);
    B.f1 = std::min(B.h, B.y1 + B.R + 1 + B.x);
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
        // the overlapped form when the band is tall enough (its workspace is reserved too);
        // one rank: the band is the whole image and runs as such (fgf_filter_band_ex)
        if (nranks > 1) {
            band_plan_overlap(B, self_guided, eps);
        } else {
            if ((rc = make_plan(B.pb, 1, rows, W, CI, CP, r, eps, s, sub))) return rc;
            B.ws_total = std::max(B.ws_total, plan_ws(B.pb, true));
        }
        return FGF_OK;
    }
    if ((rc = make_plan(B.lpB, 1, B.f1 - B.f0, B.w, CI, CP, B.R, eps, 1, FGF_SUB_NEAREST)))
        return rc;
    const size_t nc = (size_t)B.lp.NC;
    B.o_abx = B.o_lowres;                                            // a, b of the ext rows
    B.o_ab = B.o_abx + align_up(nc * B.ext_plane * sizeof(float));    // a, b rows [f0, f1)
    B.o_mean = B.o_ab + align_up(nc * B.ab_plane * sizeof(float));    // mean rows [f0, f1)
    B.ws_total = B.o_mean + align_up(nc * B.ab_plane * sizeof(float));
    if (nranks == 1) {            // one rank: the whole-image filter (fgf_filter_band_ex)
        if ((rc = make_plan(B.pb, 1, rows, W, CI, CP, r, eps, s, sub))) return rc;
        B.ws_total = std::max(B.ws_total, plan_ws(B.pb, true));
    }
    return FGF_OK;
}

// Overlapped single exchange (the default when every band holds >= 4r' + 2 low-res rows):
//   caller's stream: the low-res chain of the band's own rows as an image of its own (samples
//     read in place, any engine) -> interior maps, exact on rows [y0 + 2r', y1 - 2r') (and on
//     every row at a global image border); meanwhile on the library's comm stream:
//   comm stream: K0 compacts the 4r' own rows next to each inner band edge into an edge strip,
//     whose first / last 2r' + 1 + x rows are the halo the neighbour needs; NCCL send / recv
//     of those rows straight into the neighbours' edge strips; the low-res chain of each edge
//     strip gives the maps of rows [y0 - 1, y0 + 2r') and [y1 - 2r', y1 + 1 + x);
//   caller's stream (after both): the maps are assembled on rows [y0 - 1, y1 + 1 + x) and K4
//   writes the own rows.  The exchange runs under the interior chain; with one rank the path
//   is exactly the whole-image filter.
int band_plan_overlap(BandPlan& B, bool self_guided, double eps) {
    B.ovl = false;
    const bool up = B.row0 > 0, down = B.row0 + B.rows < B.H;   // neighbours above / below
    const int R = B.R, hb = B.y1 - B.y0;
    if (B.mode != FGF_BAND_SINGLE || hb < 4 * R + 2) return FGF_ERR_UNSUPPORTED;
    int rc = make_plan(B.pb, 1, B.rows, B.W, B.CI, B.CP, B.r_full, eps, B.s, B.sub);
    if (rc) return rc;
    if (B.pb.h != hb || B.pb.w != B.w || B.pb.R != R) return FGF_ERR_UNSUPPORTED;
    // (halo = 2r'+1+x <= 4r' rows: the rows sent lie inside the edge strips' own rows)
    B.m0 = up ? B.y0 - 1 : B.y0;
    B.m1 = down ? std::min(B.h, B.y1 + 1 + B.x) : B.y1;
    B.t0 = std::max(0, B.y0 - B.halo);
    B.t1 = B.y0 + 4 * R;
    B.b0 = B.y1 - 4 * R;
    B.b1 = std::min(B.h, B.y1 + B.halo);
    if ((rc = make_plan(B.pe_t, 1, B.t1 - B.t0, B.w, B.CI, B.CP, R, eps, 1, FGF_SUB_NEAREST)))
        return rc;
    if ((rc = make_plan(B.pe_b, 1, B.b1 - B.b0, B.w, B.CI, B.CP, R, eps, 1, FGF_SUB_NEAREST)))
        return rc;
    const size_t w = B.w, nc = B.pb.NC;
    size_t o = 0;
    B.o_slot = o; o += align_up(plan_ws(B.pb, false));
    B.o_int = o;  o += align_up(nc * hb * w * sizeof(float));
    B.o_et = o;   o += align_up((size_t)B.NPL * (B.t1 - B.t0) * w * sizeof(float));
    B.o_etw = o;  o += align_up(plan_ws(B.pe_t, false));
    B.o_etm = o;  o += align_up(nc * (B.t1 - B.t0) * w * sizeof(float));
    B.o_eb = o;   o += align_up((size_t)B.NPL * (B.b1 - B.b0) * w * sizeof(float));
    B.o_ebw = o;  o += align_up(plan_ws(B.pe_b, false));
    B.o_ebm = o;  o += align_up(nc * (B.b1 - B.b0) * w * sizeof(float));
    B.o_fin = o;  o += align_up(nc * (B.m1 - B.m0) * w * sizeof(float));
    B.ws_total = std::max(B.ws_total, o);
    B.ovl = true;
    (void)self_guided;
    return FGF_OK;
}

// Edge strips: K0 compacts the own rows [y0, t1) (top) and [b0, y1) (bottom) of every plane.
int band_ovl_prepare(const BandPlan& B, const float* I, const float* p, char* ws, cudaStream_t st) {
    const bool up = B.row0 > 0, down = B.row0 + B.rows < B.H;
    const size_t own = (size_t)B.rows * B.W, w = B.w;
    auto strip = [&](int e0, int e1, int a0, int a1, size_t off) -> int {
        // own low-res rows [a0, a1) into the strip of rows [e0, e1) at offset off
        float* ext = reinterpret_cast<float*>(ws + off);
        Plan sp{};
        sp.W = B.W; sp.s = B.s; sp.sub = B.sub; sp.w = B.w;
        sp.h = a1 - a0;
        sp.H = std::min(B.rows - (a0 - B.y0) * B.s, (a1 - a0) * B.s);
        for (int j = 0; j < B.NPL; ++j) {
            const float* src = (j < B.CI ? I + j * own : p + (j - B.CI) * own) +
                               (size_t)(a0 - B.y0) * B.s * B.W;
            float* dst = ext + (size_t)j * (e1 - e0) * w + (size_t)(a0 - e0) * w;
            int rc = launch_subsample(src, dst, 1, sp, st);
            if (rc) return rc;
        }
        return FGF_OK;
    };
    int rc;
    if (up && (rc = strip(B.t0, B.t1, B.y0, B.t1, B.o_et))) return rc;
    if (down && (rc = strip(B.b0, B.b1, B.b0, B.y1, B.o_eb))) return rc;
    return FGF_OK;
}

// Halo of plane j for the overlapped exchange: own rows [y0, y0 + halo) go up and arrive as
// the upper neighbour's rows [y1', b1'); own rows [y1 - halo, y1) go down (halo = 2r'+1+x).
Halo band_ovl_halo(const BandPlan& B, char* ws, int j) {
    const bool up = B.row0 > 0, down = B.row0 + B.rows < B.H;
    Halo hl{};
    const size_t w = B.w;
    const int H2 = B.halo;
    if (up) {
        float* et = reinterpret_cast<float*>(ws + B.o_et) + (size_t)j * (B.t1 - B.t0) * w;
        hl.n_up = (size_t)(B.y0 - B.t0) * w;
        hl.send_up = et + (size_t)(B.y0 - B.t0) * w;            // own rows [y0, y0 + H2)
        hl.recv_up = et;                                        // rows [t0, y0)
        if (B.y0 - B.t0 != H2) hl.n_up = 0;                     // (validated by the plan)
    }
    if (down) {
        float* eb = reinterpret_cast<float*>(ws + B.o_eb) + (size_t)j * (B.b1 - B.b0) * w;
        hl.n_down = (size_t)(B.b1 - B.y1) * w;
        hl.send_down = eb + (size_t)(B.y1 - H2 - B.b0) * w;     // own rows [y1 - H2, y1)
        hl.recv_down = eb + (size_t)(B.y1 - B.b0) * w;          // rows [y1, b1)
    }
    return hl;
}

// Interior: the band's own rows as an image (the whole-image low-res chain, in place).
int band_ovl_interior(const BandPlan& B, const float* I, const float* p, char* ws, cudaStream_t st) {
    return run_lowres(I, p, reinterpret_cast<float*>(ws + B.o_int), 0, 1, B.pb, ws + B.o_slot, st);
}

// Edge chains (after the exchange): maps of the edge strips.
int band_ovl_edges(const BandPlan& B, char* ws, bool self_guided, cudaStream_t st) {
    const bool up = B.row0 > 0, down = B.row0 + B.rows < B.H;
    auto chain = [&](const Plan& pe, size_t o_e, size_t o_w, size_t o_m) {
        const float* ext = reinterpret_cast<const float*>(ws + o_e);
        const size_t pl = pe.n;
        return run_coefficients(ext, self_guided ? ext : ext + B.CI * pl,
                                reinterpret_cast<float*>(ws + o_m), pe, ws + o_w,
                                plan_ws(pe, false), st);
    };
    int rc;
    if (up && (rc = chain(B.pe_t, B.o_et, B.o_etw, B.o_etm))) return rc;
    if (down && (rc = chain(B.pe_b, B.o_eb, B.o_ebw, B.o_ebm))) return rc;
    return FGF_OK;
}

// Assembly of the maps of rows [m0, m1): interior rows, then (edges = true) the edge rows.
int band_ovl_assemble(const BandPlan& B, char* ws, bool edges, cudaStream_t st) {
    const bool up = B.row0 > 0, down = B.row0 + B.rows < B.H;
    const size_t w = B.w, hm = B.m1 - B.m0, nc = B.pb.NC;
    float* fin = reinterpret_cast<float*>(ws + B.o_fin);
    auto cp = [&](const float* src, size_t src_rows, int src_r0, int dst_r0, int n) -> int {
        for (size_t m = 0; m < nc; ++m)
            if (cudaMemcpyAsync(fin + (m * hm + (dst_r0 - B.m0)) * w,
                                src + (m * src_rows + src_r0) * w, (size_t)n * w * sizeof(float),
                                cudaMemcpyDeviceToDevice, st))
                return FGF_ERR_CUDA;
        return FGF_OK;
    };
    int rc;
    if (!edges) return cp(reinterpret_cast<const float*>(ws + B.o_int), B.y1 - B.y0, 0, B.y0, B.y1 - B.y0);
    const int R = B.R;
    if (up &&
        (rc = cp(reinterpret_cast<const float*>(ws + B.o_etm), B.t1 - B.t0, B.y0 - 1 - B.t0,
                 B.y0 - 1, 2 * R + 1)))
        return rc;
    if (down &&
        (rc = cp(reinterpret_cast<const float*>(ws + B.o_ebm), B.b1 - B.b0, B.y1 - 2 * R - B.b0,
                 B.y1 - 2 * R, B.m1 - (B.y1 - 2 * R))))
        return rc;
    return FGF_OK;
}

// K4 on the own rows from the assembled maps.
int band_ovl_output(const BandPlan& B, const float* I, float* q, char* ws, cudaStream_t st) {
    Plan P{};
    P.batch = 1; P.H = B.rows; P.W = B.W; P.CI = B.CI; P.CP = B.CP; P.NC = B.pb.NC;
    P.h = B.m1 - B.m0; P.w = B.w; P.N = (size_t)B.rows * B.W; P.n = (size_t)P.h * B.w; P.TR = 32;
    const Band band{B.H, B.h, B.row0, B.m0, B.m1 - B.m0};
    return launch_output(I, reinterpret_cast<const float*>(ws + B.o_fin), q, 1, P, st, &band);
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

// Two-step exchange B geometry of a, b plane m: r'+1+x own rows each way, into [f0, y0), [y1, f1).
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
