// fgf_api.cu -- C ABI of libfgf.so (declared and documented in include/fgf.h).
//
// Host side of the hot path: argument validation (before any launch), the launch plan
// (low-res dims, r', strip and tile geometry, chunking of the batch so that each chunk's
// low-res workspace and the sample rows of I stay resident in the 126 MB L2), and the
// kernel launches of Alg. 2 on the caller's stream.
#include <mutex>

#include "fgf_host.cuh"

namespace fgf {

thread_local int g_last_launches = 0;
Profiler g_prof;

namespace {

int lowres_dim(int D, int s) { return (D + s - 1) / s; }

// R2: r' = max(1, floor(r/s + 1/2)).
int radius_lowres(int r, int s) { return std::max(1, (2 * r + s) / (2 * s)); }

int check_shape_params(int batch, int H, int W, int CI, int CP, int r, double eps, int s,
                       int sub) {
    if (batch < 1 || H < 1 || W < 1) return FGF_ERR_SHAPE;
    if (CI != 1 && CI != 3) return FGF_ERR_SHAPE;
    if (CP < 1 || CP > 4) return FGF_ERR_SHAPE;
    if (r < 1 || s < 1 || !std::isfinite(eps) || !(eps > 0.0)) return FGF_ERR_PARAM;
    if (sub != FGF_SUB_NEAREST && sub != FGF_SUB_BILINEAR) return FGF_ERR_PARAM;
    if (s > 1 && (s >= H || s >= W)) return FGF_ERR_PARAM;  // S:246, R7
    // In-image element offsets are 32-bit in the kernels (batch offsets are 64-bit).
    if ((long long)H * W * std::max(std::max(CI, CP), (CI + 1) * CP) >= (1LL << 31))
        return FGF_ERR_UNSUPPORTED;
    return FGF_OK;
}

void plan_layout(Plan& P);   // engine + workspace carve-up (below)

int make_plan(Plan& P, int batch, int H, int W, int CI, int CP, int r, double eps, int s,
              int sub) {
    int rc = check_shape_params(batch, H, W, CI, CP, r, eps, s, sub);
    if (rc) return rc;
    P.batch = batch; P.H = H; P.W = W; P.CI = CI; P.CP = CP; P.r = r; P.eps = eps; P.s = s;
    P.sub = sub;
    P.h = lowres_dim(H, s);
    P.w = lowres_dim(W, s);
    P.R = radius_lowres(r, s);
    P.NC = (CI + 1) * CP;
    P.N = (size_t)H * W;
    P.n = (size_t)P.h * P.w;

    // Strip geometry: one thread per halo column, ncol = TW + 2R <= NT.
    if (P.w <= 256) { P.nt = 256; P.TW = P.w; }
    else if (256 - 2 * P.R >= 64) { P.nt = 256; P.TW = 256 - 2 * P.R; }
    else if (P.w <= 512) { P.nt = 512; P.TW = P.w; }
    else if (512 - 2 * P.R >= 32) { P.nt = 512; P.TW = 512 - 2 * P.R; }
    else P.nt = 0;            // the strip engine cannot serve this plan (K5 may)
    P.strips = P.nt ? (P.w + P.TW - 1) / P.TW : 0;

    // Output pass: each thread walks TR full-resolution rows.
    P.TR = 32;
    P.dtype = FGF_F32;
    P.esize = 4;
    plan_layout(P);
    return P.engine == ENG_STRIP && P.nt == 0 ? FGF_ERR_UNSUPPORTED : FGF_OK;
}

// Slot layout: [planes][a, b maps][hb rings][mean maps].  need_mean: false when the caller
// provides the mean maps buffer (fgf_coefficients).
size_t plan_ws(const Plan& P, bool need_mean) {
    if (!need_mean) return std::max<size_t>(kAlign, P.ws_planes + P.ws_coef + P.ws_ring);
    return std::max<size_t>(kAlign, P.ws_slot * P.nslots);
}
size_t mean_off(const Plan& P) { return P.ws_planes + P.ws_coef + P.ws_ring; }

// Reduced-precision I/O: the engine and workspace are re-planned for the element type (the
// strip engine reads fp32 planes, so at s = 1 it needs a conversion pass into them; K13 and K5
// read the elements themselves).
int set_dtype(Plan& P, int dtype) {
    if (dtype != FGF_F32 && dtype != FGF_F16 && dtype != FGF_BF16 && dtype != FGF_U8)
        return FGF_ERR_PARAM;
    P.dtype = dtype;
    P.esize = dtype == FGF_F32 ? 4 : (dtype == FGF_U8 ? 1 : 2);
    plan_layout(P);
    return P.engine == ENG_STRIP && P.nt == 0 ? FGF_ERR_UNSUPPORTED : FGF_OK;
}

const void* elem_off(const void* base, size_t elems, const Plan& P) {
    return static_cast<const char*>(base) + elems * P.esize;
}
void* elem_off(void* base, size_t elems, const Plan& P) {
    return static_cast<char*>(base) + elems * P.esize;
}

bool overlaps(const void* a, size_t na, const void* b, size_t nb) {
    auto x = reinterpret_cast<uintptr_t>(a), y = reinterpret_cast<uintptr_t>(b);
    return x < y + nb && y < x + na;
}

bool is_device_ptr(const void* p) {
    cudaPointerAttributes at;
    if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return at.type == cudaMemoryTypeDevice || at.type == cudaMemoryTypeManaged;
}

int check_pointers(const void* I, const void* p, const void* q, const Plan& P, bool device) {
    if (!I || !p || !q) return FGF_ERR_NULL;
    if ((reinterpret_cast<uintptr_t>(I) | reinterpret_cast<uintptr_t>(p) |
         reinterpret_cast<uintptr_t>(q)) & (uintptr_t)(P.esize - 1))
        return FGF_ERR_ALIGN;
    const size_t bI = (size_t)P.batch * P.CI * P.N * P.esize;
    const size_t bp = (size_t)P.batch * P.CP * P.N * P.esize;
    if (overlaps(q, bp, I, bI) || overlaps(q, bp, p, bp)) return FGF_ERR_ALIAS;
    if (device) {
        if (!is_device_ptr(I) || !is_device_ptr(p) || !is_device_ptr(q)) return FGF_ERR_DEVICE;
    } else {
        if (is_device_ptr(I) || is_device_ptr(p) || is_device_ptr(q)) return FGF_ERR_DEVICE;
    }
    return FGF_OK;
}

// Engine choice: gray guidance at s = 1 runs the exact guided filter as ONE
// K5 kernel (Alg. 1, q written directly); gray guidance at s > 1 runs K13 for narrow
// low-res windows (r' <= 12) and K5 for wider ones; colour guidance (and what neither gray
// engine takes) runs the strip engine K1 + K3.  FGF_ENGINE=k13|wide|strip (development knob,
// FGF_DEV=1) forces an engine where it applies; FGF_LOWRES=strip is the older spelling.
int choose_engine(const Plan& P) {
    if (P.CI != 1) return ENG_STRIP;
    const bool k13 = launch_lowres_gray(LowresParams{}, P.batch, P, nullptr, true) == FGF_OK;
    WideGeom g;
    const bool wide = wide_supports(P.CP, P.dtype) && wide_geom(g, P.h, P.w, P.R, P.CP, 1, P.s == 1);
    if (const char* e = dev_env("FGF_LOWRES"))
        if (strcmp(e, "strip") == 0) return ENG_STRIP;
    const bool tiny = tiny_supports(P);
    if (const char* e = dev_env("FGF_ENGINE")) {
        if (strcmp(e, "strip") == 0) return ENG_STRIP;
        if (strcmp(e, "k13") == 0 && k13) return ENG_K13;
        if (strcmp(e, "wide") == 0 && wide) return ENG_WIDE;
        if (strcmp(e, "tiny") == 0 && tiny) return ENG_TINY;
        if (strcmp(e, "notiny") != 0 && tiny) return ENG_TINY;
    } else if (tiny) {
        return ENG_TINY;
    }
    if (P.s == 1 && wide) return ENG_WIDE;
    if (k13) return ENG_K13;
    if (wide) return ENG_WIDE;
    return ENG_STRIP;
}

// Engine and workspace per pipeline slot, recomputed from scratch (make_plan, set_dtype):
//   strip: [compact planes (s > 1 or non-fp32 I/O)] [a, b maps] [mean maps]
//   K13:   [block-mean planes (s > 1, sub = block mean)] [mean maps]
//   K5:    [block-mean planes] [mean maps, unless it writes q itself (s = 1)] [hb rings]
void plan_layout(Plan& P) {
    P.engine = choose_engine(P);
    P.fused_out = (P.engine == ENG_WIDE && P.s == 1) || P.engine == ENG_TINY;
    const bool blk = P.s > 1 && P.sub == FGF_SUB_BILINEAR;
    // (development knob FGF_WIDE_COMPACT: K5 at s > 1 reads K0-compacted nearest samples)
    const bool wcompact = P.engine == ENG_WIDE && P.s > 1 && dev_env("FGF_WIDE_COMPACT") != nullptr;
    const bool planes = P.engine == ENG_STRIP ? (P.s > 1 || P.dtype != FGF_F32) : (blk || wcompact);
    const bool coef = P.engine == ENG_STRIP;
    const bool mean = !P.fused_out || P.engine == ENG_TINY;   // K6's maps-only fallback is K13
    const size_t per_img =
        (size_t)((planes ? P.CI + P.CP : 0) + (coef ? P.NC : 0) + (mean ? P.NC : 0)) * P.n *
        sizeof(float);
    size_t target = kChunkTargetBytes;
    if (const char* e = dev_env("FGF_CHUNK_MB")) target = (size_t)atoi(e) << 20;
    P.chunk = per_img == 0 ? P.batch
                           : (int)std::max<size_t>(1, std::min<size_t>(P.batch, target / per_img));
    P.ws_planes = planes ? align_up((size_t)P.chunk * (P.CI + P.CP) * P.n * sizeof(float)) : 0;
    P.ws_coef = coef ? align_up((size_t)P.chunk * P.NC * P.n * sizeof(float)) : 0;
    P.ws_mean = mean ? align_up((size_t)P.chunk * P.NC * P.n * sizeof(float)) : 0;
    P.ws_ring = P.engine == ENG_WIDE ? wide_ring_reserve(P.R, P.CP) : 0;
    P.ws_slot = P.ws_planes + P.ws_coef + P.ws_mean + P.ws_ring;
    P.nslots = P.batch > P.chunk ? 2 : 1;
}

// Steps 1-5 for images [b0, b0+nb): writes the mean maps into `mean`.
int run_lowres(const void* I, const void* p, float* mean, int b0, int nb, const Plan& P,
               char* slot, cudaStream_t st) {
    const bool p_is_I = (I == p) && P.CI == 1 && P.CP == 1;
    const void* Ib = elem_off(I, (size_t)b0 * P.CI * P.N, P);
    const void* pb = elem_off(p, (size_t)b0 * P.CP * P.N, P);
    float* planes = reinterpret_cast<float*>(slot);
    float* coef = reinterpret_cast<float*>(slot + P.ws_planes);
    Plan Pf = P;                   // the compact planes K0 writes are fp32
    Pf.dtype = FGF_F32;
    Pf.esize = 4;
    int rc;

    // A plan whose output K5 fuses (s = 1, gray) asked here for mean maps only (fgf_coefficients,
    // the band and joint-upsampling low-res chains): K13 where it applies (needs no workspace
    // at s = 1), else K5 in its mean-maps mode.
    int eng = P.engine;
    if (P.fused_out && launch_lowres_gray(LowresParams{}, nb, P, st, true) == FGF_OK) eng = ENG_K13;
    if (eng == ENG_TINY) return FGF_ERR_UNSUPPORTED;   // (K13 always takes K6's plans)
    // Gray guidance, block-mean samples (R4): K0 compacts I', p' into fp32 planes first (and,
    // under the development knob FGF_WIDE_COMPACT, K5's nearest samples too).
    const bool blk = (P.s > 1 && P.sub == FGF_SUB_BILINEAR) ||
                     (eng == ENG_WIDE && P.s > 1 && P.ws_planes > 0 && dev_env("FGF_WIDE_COMPACT"));
    const float *Is = nullptr, *ps = nullptr;
    if (eng != ENG_STRIP && blk) {
        float* Isw = planes;
        float* psw = planes + (size_t)nb * P.n;
        if (p_is_I) {
            if ((rc = launch_subsample(Ib, Isw, nb, P, st))) return rc;
            psw = Isw;
        } else if ((rc = launch_subsample2(Ib, nb, pb, nb * P.CP, Isw, P, st))) {
            return rc;                    // I' then p' planes, psw = Isw + nb n
        }
        Is = Isw;
        ps = psw;
    }
    // Gray guidance, narrow windows: the fused K13 (nearest samples read in place).
    if (eng == ENG_K13) {
        LowresParams lp{};
        lp.h = P.h; lp.w = P.w; lp.R = P.R; lp.eps = P.eps;
        lp.k1 = P.k1; lp.k0 = P.k0;
        lp.dst = mean;
        if (blk) {
            lp.srcI = Is; lp.imgI = (long long)P.n;
            lp.srcP = ps; lp.imgP = (p_is_I ? 1LL : (long long)P.CP) * P.n; lp.planeP = (int)P.n;
            lp.row = P.w; lp.col = 1;
            return launch_lowres_gray(lp, nb, Pf, st);
        }
        // nearest (R3): sample (y, x) = I[y s][x s]; s = 1: the image itself
        lp.srcI = Ib; lp.imgI = (long long)P.N;
        lp.srcP = pb; lp.imgP = (long long)P.CP * P.N; lp.planeP = (int)P.N;
        lp.row = P.s * P.W; lp.col = P.s;
        return launch_lowres_gray(lp, nb, P, st);
    }
    // Gray guidance, wide windows: K5 in its mean-maps mode.
    if (eng == ENG_WIDE) {
        WideGeom g;
        if (!wide_geom(g, P.h, P.w, P.R, P.CP, nb, false) || g.ring_bytes > P.ws_ring)
            return FGF_ERR_UNSUPPORTED;
        WideParams wp{};
        wp.h = P.h; wp.w = P.w; wp.R = P.R; wp.eps = P.eps;
        wp.k1 = P.k1; wp.k0 = P.k0;
        wp.dst = mean;
        wp.ring = reinterpret_cast<float*>(slot + P.ws_planes + P.ws_coef);
        if (blk) {
            wp.srcI = Is; wp.imgI = (long long)P.n;
            wp.srcP = ps; wp.imgP = (p_is_I ? 1LL : (long long)P.CP) * P.n; wp.planeP = (int)P.n;
            wp.row = P.w; wp.col = 1;
            return launch_wide(wp, g, P.CP, FGF_F32, false, st);
        }
        wp.srcI = Ib; wp.imgI = (long long)P.N;
        wp.srcP = pb; wp.imgP = (long long)P.CP * P.N; wp.planeP = (int)P.N;
        wp.row = P.s * P.W; wp.col = P.s;
        return launch_wide(wp, g, P.CP, P.dtype, false, st);
    }
    if (P.nt == 0) return FGF_ERR_UNSUPPORTED;

    StripParams sp{};
    // (development knob FGF_STRIP_INPLACE: nearest fp32 samples read in place by K1, no K0)
    const bool inplace = P.s > 1 && P.sub == FGF_SUB_NEAREST && P.dtype == FGF_F32 &&
                         dev_env("FGF_STRIP_INPLACE") != nullptr;
    if (inplace) {
        sp.srcI = static_cast<const float*>(Ib); sp.imgI = (long long)P.CI * P.N; sp.planeI = (int)P.N;
        sp.srcP = static_cast<const float*>(pb); sp.imgP = (long long)P.CP * P.N; sp.planeP = (int)P.N;
        sp.row = P.s * P.W; sp.col = P.s;
    } else if (P.s > 1 || P.dtype != FGF_F32) {
        // Step 1 as its own pass (R3 nearest / R4 block mean) into compact fp32 low-res planes
        // (s = 1 with reduced-precision inputs: the conversion to fp32).
        float* Is = planes;
        float* ps = planes + (size_t)nb * P.CI * P.n;
        if (p_is_I) {
            if ((rc = launch_subsample(Ib, Is, nb * P.CI, P, st))) return rc;
            ps = Is;
        } else if ((rc = launch_subsample2(Ib, nb * P.CI, pb, nb * P.CP, Is, P, st))) {
            return rc;                    // I' then p' planes, ps = Is + nb C_I n
        }
        sp.srcI = Is; sp.imgI = (long long)P.CI * P.n; sp.planeI = (int)P.n;
        sp.srcP = ps; sp.imgP = (p_is_I ? 1LL : (long long)P.CP) * P.n; sp.planeP = (int)P.n;
        sp.row = P.w; sp.col = 1;
    } else {
        // s = 1: I' = I, p' = p; K1 reads the images directly.
        sp.srcI = static_cast<const float*>(Ib); sp.imgI = (long long)P.CI * P.N; sp.planeI = (int)P.N;
        sp.srcP = static_cast<const float*>(pb); sp.imgP = (long long)P.CP * P.N; sp.planeP = (int)P.N;
        sp.row = P.W; sp.col = 1;
    }
    sp.h = P.h; sp.w = P.w; sp.R = P.R; sp.eps = P.eps;
    sp.k1 = 1.0f; sp.k0 = 0.0f;

    // Steps 2-4: statistics + coefficients a, b.
    sp.dst = coef;
    if ((rc = launch_strip<MODE_STATS>(sp, nb, P, st))) return rc;

    // Step 5: mean_a, mean_b.
    StripParams mp{};
    mp.srcI = coef; mp.imgI = (long long)P.NC * P.n; mp.planeI = (int)P.n;
    mp.srcP = nullptr;
    mp.row = P.w; mp.col = 1;
    mp.dst = mean;
    mp.h = P.h; mp.w = P.w; mp.R = P.R; mp.eps = P.eps;
    mp.k1 = P.k1; mp.k0 = P.k0;
    return launch_strip<MODE_MEAN>(mp, nb, P, st);
}


// Per-device pipeline objects: a high-priority stream for the low-res chain and the
// fork / hand-off events.  Guarded by g_pipe_mu for the duration of an enqueue.
struct Pipe {
    bool init = false;
    cudaStream_t low = nullptr;
    cudaEvent_t fork = nullptr, done_low[2] = {nullptr, nullptr}, done_out[2] = {nullptr, nullptr};
};
std::mutex g_pipe_mu;
std::vector<Pipe> g_pipe;

int get_pipe(Pipe*& out) {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return FGF_ERR_CUDA;
    if ((int)g_pipe.size() <= dev) g_pipe.resize(dev + 1);
    Pipe& pp = g_pipe[dev];
    if (!pp.init) {
        int lo = 0, hi = 0;
        cudaDeviceGetStreamPriorityRange(&lo, &hi);
        const int prio = dev_env("FGF_LOWRES_LOWPRIO") ? lo : hi;
        if (cudaStreamCreateWithPriority(&pp.low, cudaStreamNonBlocking, prio) != cudaSuccess)
            return FGF_ERR_CUDA;
        if (cudaEventCreateWithFlags(&pp.fork, cudaEventDisableTiming)) return FGF_ERR_CUDA;
        for (int k = 0; k < 2; ++k) {
            if (cudaEventCreateWithFlags(&pp.done_low[k], cudaEventDisableTiming) ||
                cudaEventCreateWithFlags(&pp.done_out[k], cudaEventDisableTiming))
                return FGF_ERR_CUDA;
        }
        pp.init = true;
    }
    out = &pp;
    return FGF_OK;
}

// The whole filter.  Chunk j's low-res chain (K0-K3) runs on the pipeline's high-priority
// stream while the output pass K4 of chunk j-1 streams the full-resolution images on the
// caller's stream; the two workspace slots alternate.  The caller's stream is joined
// before return (it waits on the last low-res event, and all K4s are on it).
int run_all(const void* I, const void* p, void* q, const Plan& P, void* ws, size_t ws_bytes,
            cudaStream_t st) {
    if (!ws) return FGF_ERR_NULL;
    if (ws_bytes < plan_ws(P, true)) return FGF_ERR_NOMEM;
    char* base = static_cast<char*>(ws);
    if (P.engine == ENG_TINY)   // small gray image: the whole filter in one kernel, no workspace
        return launch_tiny(static_cast<const float*>(I), static_cast<const float*>(p),
                           static_cast<float*>(q), P, st);
    if (P.fused_out) {
        // s = 1, gray guidance: the exact guided filter (Alg. 1) as one K5 launch over the
        // batch -- I and p read once, q written once.
        WideGeom g;
        if (!wide_geom(g, P.h, P.w, P.R, P.CP, P.batch, true) || g.ring_bytes > P.ws_ring)
            return FGF_ERR_UNSUPPORTED;
        WideParams wp{};
        wp.h = P.h; wp.w = P.w; wp.R = P.R; wp.eps = P.eps;
        wp.k1 = P.k1; wp.k0 = P.k0;
        wp.srcI = I; wp.imgI = (long long)P.N;
        wp.srcP = p; wp.imgP = (long long)P.CP * P.N; wp.planeP = (int)P.N;
        wp.row = P.W; wp.col = 1;
        wp.q = q;
        wp.ring = reinterpret_cast<float*>(base + P.ws_planes + P.ws_coef);
        return launch_wide(wp, g, P.CP, P.dtype, true, st);
    }
    const int nchunks = (P.batch + P.chunk - 1) / P.chunk;
    if (nchunks == 1) {
        int rc = run_lowres(I, p, reinterpret_cast<float*>(base + mean_off(P)), 0, P.batch, P,
                            base, st);
        if (rc) return rc;
        // small launches (<= 16 Mi low-res samples, K13 in about one wave): K4 as a
        // programmatic dependent of K13, so its map-independent prologue and first guidance
        // rows overlap K13's tail (FGF_NO_PDL=1: a plain launch)
        Plan Po = P;
        // (the colour chain only for single-frame sizes: config 2 135.5 -> 133.3 us, while 64
        // frames of config 3 measured 1.983 -> 2.000 ms)
        const size_t lr = (size_t)P.batch * P.n;
        Po.pdl_out = ((P.engine == ENG_K13 && lr <= (16u << 20)) ||
                      (P.engine == ENG_STRIP && lr <= (1u << 20))) &&
                     dev_env("FGF_NO_PDL") == nullptr;
        return launch_output(I, reinterpret_cast<float*>(base + mean_off(P)), q, P.batch, Po, st);
    }
    std::lock_guard<std::mutex> lk(g_pipe_mu);
    Pipe* pp = nullptr;
    int rc = get_pipe(pp);
    if (rc) return rc;
    if (cudaEventRecord(pp->fork, st) || cudaStreamWaitEvent(pp->low, pp->fork, 0))
        return FGF_ERR_CUDA;
    for (int j = 0; j < nchunks; ++j) {
        const int b0 = j * P.chunk, nb = std::min(P.chunk, P.batch - b0);
        const int k = j & 1;
        char* slot = base + (size_t)k * P.ws_slot;
        float* mean = reinterpret_cast<float*>(slot + mean_off(P));
        // The slot is free once the output pass of chunk j-2 has read its mean maps.
        if (j >= 2 && cudaStreamWaitEvent(pp->low, pp->done_out[k], 0)) return FGF_ERR_CUDA;
        if ((rc = run_lowres(I, p, mean, b0, nb, P, slot, pp->low))) return rc;
        if (cudaEventRecord(pp->done_low[k], pp->low) || cudaStreamWaitEvent(st, pp->done_low[k], 0))
            return FGF_ERR_CUDA;
        if ((rc = launch_output(elem_off(I, (size_t)b0 * P.CI * P.N, P), mean,
                                elem_off(q, (size_t)b0 * P.CP * P.N, P), nb, P, st)))
            return rc;
        if (cudaEventRecord(pp->done_out[k], st)) return FGF_ERR_CUDA;
    }
    return FGF_OK;
}

// Steps 1-5 into a caller buffer (fgf_coefficients), on the caller's stream.
int run_coefficients(const void* I, const void* p, float* mean_out, const Plan& P, void* ws,
                     size_t ws_bytes, cudaStream_t st) {
    if (!ws) return FGF_ERR_NULL;
    if (ws_bytes < plan_ws(P, false)) return FGF_ERR_NOMEM;
    for (int b0 = 0; b0 < P.batch; b0 += P.chunk) {
        const int nb = std::min(P.chunk, P.batch - b0);
        int rc = run_lowres(I, p, mean_out + (size_t)b0 * P.NC * P.n, b0, nb, P,
                            static_cast<char*>(ws), st);
        if (rc) return rc;
    }
    return FGF_OK;
}

// Internal grow-only workspace for fgf_filter(), one per device.
struct DevWs {
    void* ptr = nullptr;
    size_t bytes = 0;
};
std::mutex g_ws_mu;
std::vector<DevWs> g_ws;

// Host-buffer pipeline state (fgf_filter_host), one per device.
constexpr int kHostBands = 8;
struct HostPipe {
    float* dbuf[2] = {nullptr, nullptr};
    size_t dbytes = 0;
    void* ws = nullptr;
    size_t wsbytes = 0;
    cudaStream_t s_h2d = nullptr, s_comp = nullptr, s_d2h = nullptr;
    cudaEvent_t ev_in[2], ev_done[2], ev_free[2];
    cudaEvent_t ev_bin[kHostBands], ev_bout[kHostBands];   // single-frame row-band pipeline
    bool init = false;
};
std::mutex g_host_mu;
std::vector<HostPipe> g_host;

// Band path: the library's comm stream (edge strips, NCCL halo, edge chains) and its events.
struct BandStreams {
    bool init = false;
    cudaStream_t comm = nullptr;
    cudaEvent_t fork = nullptr, interior = nullptr, edges = nullptr;
};
std::mutex g_band_mu;
std::vector<BandStreams> g_band;

int get_band_streams(BandStreams*& out) {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return FGF_ERR_CUDA;
    if ((int)g_band.size() <= dev) g_band.resize(dev + 1);
    BandStreams& b = g_band[dev];
    if (!b.init) {
        int lo = 0, hi = 0;
        cudaDeviceGetStreamPriorityRange(&lo, &hi);
        if (cudaStreamCreateWithPriority(&b.comm, cudaStreamNonBlocking, hi) ||
            cudaEventCreateWithFlags(&b.fork, cudaEventDisableTiming) ||
            cudaEventCreateWithFlags(&b.interior, cudaEventDisableTiming) ||
            cudaEventCreateWithFlags(&b.edges, cudaEventDisableTiming))
            return FGF_ERR_CUDA;
        b.init = true;
    }
    out = &b;
    return FGF_OK;
}

// ---- CUDA-graph cache for small calls (verdict r1: single-image latency).  A call of at most
// kGraphMaxPixels output pixels whose arguments (pointers, sizes, parameters, stream,
// workspace) repeat an earlier call is replayed from a graph captured on its second occurrence:
// no per-launch host overhead, no validation queries, no inter-kernel launch gaps.  Not used
// on the legacy default stream (not capturable), with per-launch profiling on, with the
// development knobs (FGF_DEV=1) or FGF_DEBUG_SYNC, or with FGF_GRAPHS=0.
constexpr size_t kGraphMaxPixels = 32u << 20;
constexpr int kGraphSlots = 32;

struct GraphKey {
    const void *I, *p, *q, *ws;
    size_t ws_bytes;
    void* stream;
    int batch, H, W, CI, CP, r, s, sub, dtype, dev, kind;
    double eps, gain;
    bool operator==(const GraphKey& o) const { return memcmp(this, &o, sizeof(GraphKey)) == 0; }
};
struct GraphEntry {
    GraphKey key;
    cudaGraphExec_t exec = nullptr;   // nullptr: seen once, not captured yet
    int launches = 0;
    unsigned long long used = 0;
};
std::mutex g_graph_mu;
std::vector<GraphEntry> g_graphs;
unsigned long long g_graph_clock = 0;

GraphKey graph_key(int kind, const void* I, const void* p, const void* q, const Plan& P,
                   double gain, const void* ws, size_t ws_bytes, cudaStream_t st) {
    GraphKey k;
    memset(&k, 0, sizeof(k));   // padding bytes take part in the comparison
    k.I = I; k.p = p; k.q = q; k.ws = ws; k.ws_bytes = ws_bytes; k.stream = st;
    k.batch = P.batch; k.H = P.H; k.W = P.W; k.CI = P.CI; k.CP = P.CP; k.r = P.r; k.s = P.s;
    k.sub = P.sub; k.dtype = P.dtype; k.kind = kind; k.eps = P.eps; k.gain = gain;
    cudaGetDevice(&k.dev);
    return k;
}

bool graph_eligible(const Plan& P, cudaStream_t st) {
    if (st == nullptr || st == cudaStreamLegacy || st == cudaStreamPerThread) return false;
    if ((size_t)P.batch * P.N > kGraphMaxPixels || g_prof.on || debug_sync()) return false;
    if (const char* d = getenv("FGF_DEV"))
        if (atoi(d) != 0) return false;
    if (const char* e = getenv("FGF_GRAPHS"))
        if (atoi(e) == 0) return false;
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    if (cudaStreamIsCapturing(st, &cs) != cudaSuccess || cs != cudaStreamCaptureStatusNone) {
        cudaGetLastError();
        return false;                  // the caller is capturing: enqueue normally
    }
    return true;
}

// validate: the pointer checks (run on first sight only); enqueue: the launches.
template <typename V, typename F>
int run_cached(const GraphKey& key, cudaStream_t st, V&& validate, F&& enqueue) {
    std::lock_guard<std::mutex> lk(g_graph_mu);
    GraphEntry* e = nullptr;
    for (auto& x : g_graphs)
        if (x.key == key) e = &x;
    if (e && e->exec) {
        e->used = ++g_graph_clock;
        g_last_launches = e->launches;
        return cudaGraphLaunch(e->exec, st) == cudaSuccess ? FGF_OK : FGF_ERR_CUDA;
    }
    int rc = validate();
    if (rc) return rc;
    if (!e) {                          // first sight: run eagerly, remember the arguments
        rc = enqueue();
        if (rc) return rc;
        if ((int)g_graphs.size() >= kGraphSlots) {
            auto lru = std::min_element(g_graphs.begin(), g_graphs.end(),
                                        [](const GraphEntry& a, const GraphEntry& b) { return a.used < b.used; });
            if (lru->exec) cudaGraphExecDestroy(lru->exec);
            g_graphs.erase(lru);
        }
        GraphEntry ne;
        ne.key = key;
        ne.used = ++g_graph_clock;
        g_graphs.push_back(ne);
        return FGF_OK;
    }
    // second sight: capture the same launches, instantiate, replay
    cudaGraph_t graph = nullptr;
    if (cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal) != cudaSuccess) {
        cudaGetLastError();
        return enqueue();
    }
    rc = enqueue();
    const int launches = g_last_launches;
    const cudaError_t ce = cudaStreamEndCapture(st, &graph);
    cudaGraphExec_t exec = nullptr;
    if (rc || ce != cudaSuccess || !graph ||
        cudaGraphInstantiate(&exec, graph, 0) != cudaSuccess) {
        cudaGetLastError();
        if (graph) cudaGraphDestroy(graph);
        if (rc) return rc;
        return enqueue();              // capture failed: the launches were not run yet
    }
    cudaGraphDestroy(graph);
    e->exec = exec;
    e->launches = launches;
    e->used = ++g_graph_clock;
    g_last_launches = launches;
    return cudaGraphLaunch(exec, st) == cudaSuccess ? FGF_OK : FGF_ERR_CUDA;
}

}  // namespace
}  // namespace fgf

#include "fgf_band.cuh"

using namespace fgf;

extern "C" {

const char* fgf_version(void) { return "fgf-b200 0.2 (sm_100a)"; }

int fgf_last_launch_count(void) { return g_last_launches; }

int fgf_profile_enable(int on) {
    g_prof.clear();
    g_prof.on = on != 0;
    return FGF_OK;
}

int fgf_profile_read(double* ms, int* launches, int max_kinds) {
    const int nk = std::min<int>(max_kinds, NKIND);
    for (int k = 0; k < nk; ++k) {
        if (ms) ms[k] = 0.0;
        if (launches) launches[k] = 0;
    }
    for (auto& r : g_prof.recs) {
        if (cudaEventSynchronize(r.b) != cudaSuccess) return -FGF_ERR_CUDA;
        float t = 0.f;
        if (cudaEventElapsedTime(&t, r.a, r.b) != cudaSuccess) return -FGF_ERR_CUDA;
        if (r.kind < nk) {
            if (ms) ms[r.kind] += t;
            if (launches) launches[r.kind] += 1;
        }
    }
    g_prof.clear();
    return nk;
}

const char* fgf_status_str(int status) {
    switch (status) {
        case FGF_OK: return "ok";
        case FGF_ERR_PARAM: return "invalid parameter (r, eps, s, sub_mode)";
        case FGF_ERR_SHAPE: return "invalid shape (batch, H, W, C_I, C_p)";
        case FGF_ERR_NULL: return "null pointer";
        case FGF_ERR_ALIAS: return "output overlaps an input";
        case FGF_ERR_ALIGN: return "pointer not 4-byte aligned";
        case FGF_ERR_CUDA: return "CUDA error";
        case FGF_ERR_NOMEM: return "workspace too small or allocation failed";
        case FGF_ERR_NCCL: return "NCCL error";
        case FGF_ERR_UNSUPPORTED: return "unsupported geometry (no engine serves it)";
        case FGF_ERR_DEVICE: return "pointer is in the wrong memory space";
    }
    return "unknown status";
}

size_t fgf_workspace_bytes(int batch, int H, int W, int C_I, int C_p, int r, int s) {
    // The larger of the two subsampling modes (block mean needs the I', p' planes).
    Plan P0, P1;
    if (make_plan(P0, batch, H, W, C_I, C_p, r, 1.0, s, FGF_SUB_NEAREST)) return 0;
    if (make_plan(P1, batch, H, W, C_I, C_p, r, 1.0, s, FGF_SUB_BILINEAR)) return 0;
    return std::max(plan_ws(P0, true), plan_ws(P1, true));
}

size_t fgf_workspace_bytes_ex(int batch, int H, int W, int C_I, int C_p, int r, int s, int dtype) {
    Plan P0, P1;
    if (make_plan(P0, batch, H, W, C_I, C_p, r, 1.0, s, FGF_SUB_NEAREST)) return 0;
    if (make_plan(P1, batch, H, W, C_I, C_p, r, 1.0, s, FGF_SUB_BILINEAR)) return 0;
    if (set_dtype(P0, dtype) || set_dtype(P1, dtype)) return 0;
    return std::max(plan_ws(P0, true), plan_ws(P1, true));
}

int fgf_filter_ex_ws(const void* I, const void* p, void* q, int batch, int H, int W, int C_I,
                     int C_p, int r, double eps, int s, int sub_mode, int dtype, void* workspace,
                     size_t ws_bytes, void* cuda_stream) {
    g_last_launches = 0;
    Plan P;
    int rc = make_plan(P, batch, H, W, C_I, C_p, r, eps, s, sub_mode);
    if (rc) return rc;
    if ((rc = set_dtype(P, dtype))) return rc;
    if (dtype != FGF_F32 && !(C_I * 10 + C_p == 11 || C_I * 10 + C_p == 31 || C_I * 10 + C_p == 33))
        return FGF_ERR_UNSUPPORTED;
    cudaStream_t st = static_cast<cudaStream_t>(cuda_stream);
    auto validate = [&] { return check_pointers(I, p, q, P, true); };
    auto enqueue = [&] { return run_all(I, p, q, P, workspace, ws_bytes, st); };
    if (graph_eligible(P, st))
        return run_cached(graph_key(0, I, p, q, P, 0.0, workspace, ws_bytes, st), st, validate, enqueue);
    if ((rc = validate())) return rc;
    return enqueue();
}

int fgf_filter_ws(const float* I, const float* p, float* q, int batch, int H, int W, int C_I,
                  int C_p, int r, double eps, int s, int sub_mode, void* workspace,
                  size_t ws_bytes, void* cuda_stream) {
    g_last_launches = 0;
    Plan P;
    int rc = make_plan(P, batch, H, W, C_I, C_p, r, eps, s, sub_mode);
    if (rc) return rc;
    cudaStream_t st = static_cast<cudaStream_t>(cuda_stream);
    auto validate = [&] { return check_pointers(I, p, q, P, true); };
    auto enqueue = [&] { return run_all(I, p, q, P, workspace, ws_bytes, st); };
    if (graph_eligible(P, st))
        return run_cached(graph_key(0, I, p, q, P, 0.0, workspace, ws_bytes, st), st, validate, enqueue);
    if ((rc = validate())) return rc;
    return enqueue();
}

int fgf_nccl_unique_id(void* id_out) {
    if (!id_out) return FGF_ERR_NULL;
    const Nccl* n = nccl();
    if (!n) return FGF_ERR_NCCL;
    return n->getUniqueId(static_cast<ncclUniqueId*>(id_out)) == ncclSuccess ? FGF_OK : FGF_ERR_NCCL;
}

int fgf_nccl_comm_init(void** comm_out, const void* id, int rank, int nranks) {
    if (!comm_out || !id) return FGF_ERR_NULL;
    if (nranks < 1 || rank < 0 || rank >= nranks) return FGF_ERR_PARAM;
    const Nccl* n = nccl();
    if (!n) return FGF_ERR_NCCL;
    ncclUniqueId uid;
    memcpy(&uid, id, sizeof(uid));
    ncclComm_t c = nullptr;
    if (n->commInitRank(&c, nranks, uid, rank) != ncclSuccess) return FGF_ERR_NCCL;
    *comm_out = c;
    return FGF_OK;
}

int fgf_nccl_check(void* comm) {
    if (!comm) return FGF_ERR_NULL;
    const Nccl* n = nccl();
    if (!n || !n->commGetAsyncError) return FGF_ERR_NCCL;
    ncclResult_t async = ncclSuccess;
    if (n->commGetAsyncError(static_cast<ncclComm_t>(comm), &async) != ncclSuccess) return FGF_ERR_NCCL;
    return async == ncclSuccess || async == ncclInProgress ? FGF_OK : FGF_ERR_NCCL;
}

int fgf_nccl_comm_destroy(void* comm) {
    if (!comm) return FGF_ERR_NULL;
    const Nccl* n = nccl();
    if (!n) return FGF_ERR_NCCL;
    return n->commDestroy(static_cast<ncclComm_t>(comm)) == ncclSuccess ? FGF_OK : FGF_ERR_NCCL;
}

int fgf_band_geometry(int H, int W, int r, int s, int nranks, int rank, int* out) {
    if (!out) return FGF_ERR_NULL;
    if (H < 1 || W < 1) return FGF_ERR_SHAPE;
    if (r < 1 || s < 1 || nranks < 1 || rank < 0 || rank >= nranks) return FGF_ERR_PARAM;
    const int h = lowres_dim(H, s), w = lowres_dim(W, s), R = radius_lowres(r, s);
    // 2r'+1 rows, plus one when h s != H (the map scale h / H > 1 / s: a band's last rows
    // upsample from up to low-res row y1 + 1; fgf_band.cuh)
    const int halo = 2 * R + 1 + ((long long)h * s != H ? 1 : 0);
    // every band must hold a whole single-exchange halo, unless it is alone
    for (int k = 0; k < nranks && nranks > 1; ++k)
        if ((int)((long long)(k + 1) * h / nranks) - (int)((long long)k * h / nranks) < halo)
            return FGF_ERR_PARAM;
    const int y0 = (int)((long long)rank * h / nranks), y1 = (int)((long long)(rank + 1) * h / nranks);
    const int g[10] = {h, w, R, halo, y0, y1, y0 * s, std::min(H, y1 * s), std::max(0, y0 - halo),
                       std::min(h, y1 + halo)};
    memcpy(out, g, sizeof(g));
    return FGF_OK;
}

size_t fgf_band_workspace_bytes(int H_total, int W, int row0, int rows, int C_I, int C_p, int r,
                                int s, int nranks) {
    // The larger of the exchange modes this band admits (two-step accepts narrower bands:
    // r'+1 low-res rows instead of 2r'+1) and of the two subsampling modes (the band's own
    // chain may need the I', p' planes under the block mean); 0 only when no mode accepts the
    // band.
    size_t best = 0;
    for (int mode : {FGF_BAND_SINGLE, FGF_BAND_TWO_STEP})
        for (int sub : {FGF_SUB_NEAREST, FGF_SUB_BILINEAR}) {
            BandPlan B;
            if (band_plan(B, H_total, W, row0, rows, C_I, C_p, r, 1.0, s, sub, nranks, false,
                          mode) == FGF_OK)
                best = std::max(best, B.ws_total);
        }
    return best;
}

int fgf_filter_band(const float* I_band, const float* p_band, float* q_band, int H_total, int W,
                    int row0, int rows, int C_I, int C_p, int r, double eps, int s, int sub_mode,
                    void* nccl_comm, int rank, int nranks, void* workspace, size_t ws_bytes,
                    void* cuda_stream) {
    return fgf_filter_band_ex(I_band, p_band, q_band, H_total, W, row0, rows, C_I, C_p, r, eps, s,
                              sub_mode, FGF_BAND_SINGLE, nccl_comm, rank, nranks, workspace,
                              ws_bytes, cuda_stream);
}

int fgf_filter_band_ex(const float* I_band, const float* p_band, float* q_band, int H_total,
                       int W, int row0, int rows, int C_I, int C_p, int r, double eps, int s,
                       int sub_mode, int mode, void* nccl_comm, int rank, int nranks,
                       void* workspace, size_t ws_bytes, void* cuda_stream) {
    g_last_launches = 0;
    if (nranks < 1 || rank < 0 || rank >= nranks) return FGF_ERR_PARAM;
    const bool self = I_band == p_band && C_I == 1 && C_p == 1;
    BandPlan B;
    int rc = band_plan(B, H_total, W, row0, rows, C_I, C_p, r, eps, s, sub_mode, nranks, self,
                       mode);
    if (rc) return rc;
    if (!I_band || !p_band || !q_band || !workspace) return FGF_ERR_NULL;
    if (nranks > 1 && !nccl_comm) return FGF_ERR_NULL;
    if ((reinterpret_cast<uintptr_t>(I_band) | reinterpret_cast<uintptr_t>(p_band) |
         reinterpret_cast<uintptr_t>(q_band)) & 3u)
        return FGF_ERR_ALIGN;
    const size_t own = (size_t)rows * W * 4;
    if (overlaps(q_band, C_p * own, I_band, C_I * own) || overlaps(q_band, C_p * own, p_band, C_p * own))
        return FGF_ERR_ALIAS;
    if (!is_device_ptr(I_band) || !is_device_ptr(p_band) || !is_device_ptr(q_band) ||
        !is_device_ptr(workspace))
        return FGF_ERR_DEVICE;
    if (ws_bytes < B.ws_total) return FGF_ERR_NOMEM;
    cudaStream_t st = static_cast<cudaStream_t>(cuda_stream);
    char* ws = static_cast<char*>(workspace);
    // one NCCL group: every plane's halo rows to / from rank-1 and rank+1
    auto nccl_exchange = [&](int planes, auto&& halo_of, cudaStream_t cs) -> int {
        const Nccl* n = nccl();
        if (!n) return FGF_ERR_NCCL;
        ncclComm_t comm = static_cast<ncclComm_t>(nccl_comm);
        if (n->groupStart() != ncclSuccess) return FGF_ERR_NCCL;
        ncclResult_t e = ncclSuccess;
        for (int j = 0; j < planes && e == ncclSuccess; ++j) {
            const Halo hl = halo_of(j);
            if (hl.n_up) {
                e = n->send(hl.send_up, hl.n_up, ncclFloat32, rank - 1, comm, cs);
                if (e == ncclSuccess) e = n->recv(hl.recv_up, hl.n_up, ncclFloat32, rank - 1, comm, cs);
            }
            if (hl.n_down && e == ncclSuccess) {
                e = n->send(hl.send_down, hl.n_down, ncclFloat32, rank + 1, comm, cs);
                if (e == ncclSuccess) e = n->recv(hl.recv_down, hl.n_down, ncclFloat32, rank + 1, comm, cs);
            }
        }
        if (n->groupEnd() != ncclSuccess || e != ncclSuccess) return FGF_ERR_NCCL;
        return FGF_OK;
    };
    if (nranks == 1)   // one band = the whole image: the whole-image filter itself
        return run_all(I_band, p_band, q_band, B.pb, ws, ws_bytes, st);
    if (B.ovl) {
        // overlapped single exchange (fgf_band.cuh): interior chain on the caller's stream,
        // edge strips + NCCL halo + edge chains on the library's comm stream
        std::lock_guard<std::mutex> lk(g_band_mu);
        BandStreams* bs = nullptr;
        if ((rc = get_band_streams(bs))) return rc;
        const int launches0 = g_last_launches;
        if (cudaEventRecord(bs->fork, st) || cudaStreamWaitEvent(bs->comm, bs->fork, 0)) return FGF_ERR_CUDA;
        if ((rc = band_ovl_prepare(B, I_band, p_band, ws, bs->comm))) return rc;
        if ((rc = nccl_exchange(B.NPL, [&](int j) { return band_ovl_halo(B, ws, j); }, bs->comm)))
            return rc;
        if ((rc = band_ovl_interior(B, I_band, p_band, ws, st))) return rc;
        if ((rc = band_ovl_assemble(B, ws, false, st))) return rc;
        if (cudaEventRecord(bs->interior, st)) return FGF_ERR_CUDA;
        if ((rc = band_ovl_edges(B, ws, self, bs->comm))) return rc;
        if (cudaStreamWaitEvent(bs->comm, bs->interior, 0)) return FGF_ERR_CUDA;
        if ((rc = band_ovl_assemble(B, ws, true, bs->comm))) return rc;
        if (cudaEventRecord(bs->edges, bs->comm) || cudaStreamWaitEvent(st, bs->edges, 0))
            return FGF_ERR_CUDA;
        rc = band_ovl_output(B, I_band, q_band, ws, st);
        (void)launches0;
        return rc;
    }
    if ((rc = band_prepare(B, I_band, p_band, ws, st))) return rc;
    if ((rc = nccl_exchange(B.NPL, [&](int j) { return band_halo(B, ws, j, rank, nranks); }, st)))
        return rc;                                                      // I', p' (exchange A)
    if (B.mode == FGF_BAND_TWO_STEP) {
        if ((rc = band_stats_ab(B, ws, st, self))) return rc;
        if ((rc = nccl_exchange(B.lp.NC, [&](int j) { return band_halo_ab(B, ws, j, rank, nranks); }, st)))
            return rc;                                                  // a, b (exchange B)
    }
    return band_finish(B, I_band, q_band, ws, st, self);
}

size_t fgf_bands_loopback_workspace_bytes(int H, int W, int C_I, int C_p, int r, int s,
                                          int nranks) {
    // per band: the larger of the exchange modes the band admits (as fgf_band_workspace_bytes)
    if (nranks < 1 || s < 1 || H < 1 || W < 1) return 0;
    const int h = lowres_dim(H, s);
    size_t tot = 0;
    for (int k = 0; k < nranks; ++k) {
        const int y0 = (int)((long long)k * h / nranks), y1 = (int)((long long)(k + 1) * h / nranks);
        const int row0 = y0 * s, rows = std::min(H, y1 * s) - row0;
        if (rows < 1) return 0;
        const size_t b = fgf_band_workspace_bytes(H, W, row0, rows, C_I, C_p, r, s, nranks);
        if (b == 0) return 0;
        tot += b + 2 * align_up((size_t)(C_I + 2 * C_p) * rows * W * 4);
    }
    return tot;
}

int fgf_filter_bands_loopback(const float* I, const float* p, float* q, int H, int W, int C_I,
                              int C_p, int r, double eps, int s, int sub_mode, int mode,
                              int nranks, void* workspace, size_t ws_bytes, void* cuda_stream) {
    g_last_launches = 0;
    if (nranks < 1) return FGF_ERR_PARAM;
    Plan P0;
    int rc = make_plan(P0, 1, H, W, C_I, C_p, r, eps, s, sub_mode);
    if (rc) return rc;
    if ((rc = check_pointers(I, p, q, P0, true))) return rc;
    if (!workspace) return FGF_ERR_NULL;
    if (ws_bytes < fgf_bands_loopback_workspace_bytes(H, W, C_I, C_p, r, s, nranks))
        return FGF_ERR_NOMEM;
    cudaStream_t st = static_cast<cudaStream_t>(cuda_stream);
    const bool self = I == p && C_I == 1 && C_p == 1;
    const int h = P0.h;
    std::vector<BandPlan> Bs(nranks);
    std::vector<char*> wss(nranks);
    std::vector<float*> Ib(nranks), pb(nranks), qb(nranks);
    char* cur = static_cast<char*>(workspace);
    int launches = 0;
    for (int k = 0; k < nranks; ++k) {
        const int y0 = (int)((long long)k * h / nranks), y1 = (int)((long long)(k + 1) * h / nranks);
        const int row0 = y0 * s, rows = std::min(H, y1 * s) - row0;
        if ((rc = band_plan(Bs[k], H, W, row0, rows, C_I, C_p, r, eps, s, sub_mode, nranks, self,
                            mode)))
            return rc;
        wss[k] = cur;
        // the workspace layout reserves what the size query reserved for this band
        const size_t wsb = fgf_band_workspace_bytes(H, W, row0, rows, C_I, C_p, r, s, nranks);
        if (wsb < Bs[k].ws_total) return FGF_ERR_NOMEM;
        cur += wsb;
        // the band's own rows, contiguous per plane, as a rank would hold them
        Ib[k] = reinterpret_cast<float*>(cur);
        pb[k] = self ? Ib[k] : Ib[k] + (size_t)C_I * rows * W;
        qb[k] = Ib[k] + (size_t)(C_I + C_p) * rows * W;
        cur += 2 * align_up((size_t)(C_I + 2 * C_p) * rows * W * 4);
        for (int j = 0; j < C_I; ++j)
            if (cudaMemcpyAsync(Ib[k] + (size_t)j * rows * W, I + ((size_t)j * H + row0) * W,
                                (size_t)rows * W * 4, cudaMemcpyDeviceToDevice, st))
                return FGF_ERR_CUDA;
        if (!self)
            for (int j = 0; j < C_p; ++j)
                if (cudaMemcpyAsync(pb[k] + (size_t)j * rows * W, p + ((size_t)j * H + row0) * W,
                                    (size_t)rows * W * 4, cudaMemcpyDeviceToDevice, st))
                    return FGF_ERR_CUDA;
    }
    // the overlapped single exchange when every band takes it (as fgf_filter_band_ex)
    bool use_ovl = mode == FGF_BAND_SINGLE && nranks > 1;
    for (int k = 0; k < nranks; ++k) use_ovl = use_ovl && Bs[k].ovl;
    for (int k = 0; k < nranks; ++k) {
        if ((rc = use_ovl ? band_ovl_prepare(Bs[k], Ib[k], pb[k], wss[k], st)
                          : band_prepare(Bs[k], Ib[k], pb[k], wss[k], st)))
            return rc;
        launches += g_last_launches;
        g_last_launches = 0;
    }
    // the exchanges, rank k <-> k+1, with the same halo geometry the NCCL path sends
    // (0: I', p' of the compacting single / two-step forms, 1: a, b, 2: overlapped form)
    auto exchange = [&](int kind) -> int {
        for (int k = 0; k + 1 < nranks; ++k) {
            const int planes = kind == 1 ? Bs[k].lp.NC : Bs[k].NPL;
            for (int j = 0; j < planes; ++j) {
                auto halo = [&](int kk) {
                    return kind == 2 ? band_ovl_halo(Bs[kk], wss[kk], j)
                         : kind == 1 ? band_halo_ab(Bs[kk], wss[kk], j, kk, nranks)
                                     : band_halo(Bs[kk], wss[kk], j, kk, nranks);
                };
                const Halo a = halo(k), b = halo(k + 1);
                if (a.n_down != b.n_up) return FGF_ERR_PARAM;   // both sides agree on the depth
                if (cudaMemcpyAsync(a.recv_down, b.send_up, b.n_up * 4, cudaMemcpyDeviceToDevice, st) ||
                    cudaMemcpyAsync(b.recv_up, a.send_down, a.n_down * 4, cudaMemcpyDeviceToDevice, st))
                    return FGF_ERR_CUDA;
            }
        }
        return FGF_OK;
    };
    if (use_ovl) {
        if ((rc = exchange(2))) return rc;
        for (int k = 0; k < nranks; ++k) {
            if ((rc = band_ovl_interior(Bs[k], Ib[k], pb[k], wss[k], st)) ||
                (rc = band_ovl_assemble(Bs[k], wss[k], false, st)) ||
                (rc = band_ovl_edges(Bs[k], wss[k], self, st)) ||
                (rc = band_ovl_assemble(Bs[k], wss[k], true, st)) ||
                (rc = band_ovl_output(Bs[k], Ib[k], qb[k], wss[k], st)))
                return rc;
            launches += g_last_launches;
            g_last_launches = 0;
            for (int j = 0; j < C_p; ++j)
                if (cudaMemcpyAsync(q + ((size_t)j * H + Bs[k].row0) * W, qb[k] + (size_t)j * Bs[k].rows * W,
                                    (size_t)Bs[k].rows * W * 4, cudaMemcpyDeviceToDevice, st))
                    return FGF_ERR_CUDA;
        }
        g_last_launches = launches;
        return FGF_OK;
    }
    if ((rc = exchange(0))) return rc;
    if (mode == FGF_BAND_TWO_STEP) {
        for (int k = 0; k < nranks; ++k) {
            if ((rc = band_stats_ab(Bs[k], wss[k], st, self))) return rc;
            launches += g_last_launches;
            g_last_launches = 0;
        }
        if ((rc = exchange(1))) return rc;
    }
    for (int k = 0; k < nranks; ++k) {
        if ((rc = band_finish(Bs[k], Ib[k], qb[k], wss[k], st, self))) return rc;
        launches += g_last_launches;
        g_last_launches = 0;
        for (int j = 0; j < C_p; ++j)
            if (cudaMemcpyAsync(q + ((size_t)j * H + Bs[k].row0) * W, qb[k] + (size_t)j * Bs[k].rows * W,
                                (size_t)Bs[k].rows * W * 4, cudaMemcpyDeviceToDevice, st))
                return FGF_ERR_CUDA;
    }
    g_last_launches = launches;
    return FGF_OK;
}

// ---- joint upsampling (R18): p given at low resolution
struct JointPlan {
    Plan P;                  // the full-resolution plan (I, q)
    Plan L;                  // the s = 1 plan on the low-res planes, radius r'
    size_t o_planes, o_lowres, o_mean, total;
};

int joint_plan(JointPlan& J, int batch, int H, int W, int CI, int CP, int r, double eps, int s,
               int sub) {
    int rc = make_plan(J.P, batch, H, W, CI, CP, r, eps, s, sub);
    if (rc) return rc;
    if ((rc = make_plan(J.L, batch, J.P.h, J.P.w, CI, CP, J.P.R, eps, 1, FGF_SUB_NEAREST)))
        return rc;
    J.o_planes = 0;
    J.o_lowres = align_up((size_t)batch * CI * J.P.n * sizeof(float));
    J.o_mean = J.o_lowres + align_up(plan_ws(J.L, false));     // reused chunk by chunk
    J.total = J.o_mean + align_up((size_t)batch * J.P.NC * J.P.n * sizeof(float));
    return FGF_OK;
}

size_t fgf_joint_workspace_bytes(int batch, int H, int W, int C_I, int C_p, int r, int s) {
    JointPlan J;
    if (joint_plan(J, batch, H, W, C_I, C_p, r, 1.0, s, FGF_SUB_NEAREST)) return 0;
    JointPlan J2;
    if (joint_plan(J2, batch, H, W, C_I, C_p, r, 1.0, s, FGF_SUB_BILINEAR)) return 0;
    return std::max(J.total, J2.total);
}

int fgf_filter_joint_ws(const float* I, const float* p_low, float* q, int batch, int H, int W,
                        int C_I, int C_p, int r, double eps, int s, int sub_mode,
                        void* workspace, size_t ws_bytes, void* cuda_stream) {
    g_last_launches = 0;
    JointPlan J;
    int rc = joint_plan(J, batch, H, W, C_I, C_p, r, eps, s, sub_mode);
    if (rc) return rc;
    const Plan& P = J.P;
    if (!I || !p_low || !q || !workspace) return FGF_ERR_NULL;
    if ((reinterpret_cast<uintptr_t>(I) | reinterpret_cast<uintptr_t>(p_low) |
         reinterpret_cast<uintptr_t>(q)) & 3u)
        return FGF_ERR_ALIGN;
    const size_t bq = (size_t)batch * C_p * P.N * 4;
    if (overlaps(q, bq, I, (size_t)batch * C_I * P.N * 4) ||
        overlaps(q, bq, p_low, (size_t)batch * C_p * P.n * 4))
        return FGF_ERR_ALIAS;
    if (!is_device_ptr(I) || !is_device_ptr(p_low) || !is_device_ptr(q) || !is_device_ptr(workspace))
        return FGF_ERR_DEVICE;
    if (ws_bytes < J.total) return FGF_ERR_NOMEM;
    cudaStream_t st = static_cast<cudaStream_t>(cuda_stream);
    char* ws = static_cast<char*>(workspace);
    float* Is = reinterpret_cast<float*>(ws + J.o_planes);
    float* mean = reinterpret_cast<float*>(ws + J.o_mean);
    // step 1 for I only (p' is given), steps 2-5 on (I', p'), steps 6-7 with the full-res I
    if ((rc = launch_subsample(I, Is, batch * C_I, P, st))) return rc;
    int launches = g_last_launches;
    if ((rc = run_coefficients(Is, p_low, mean, J.L, ws + J.o_lowres, J.o_mean - J.o_lowres, st)))
        return rc;
    launches += g_last_launches;
    g_last_launches = 0;
    rc = launch_output(I, mean, q, batch, P, st);
    g_last_launches += launches;
    return rc;
}

int fgf_enhance_ws(const float* I, float* out, int batch, int H, int W, int C, int r,
                   double eps, int s, int sub_mode, double gain, void* workspace,
                   size_t ws_bytes, void* cuda_stream) {
    g_last_launches = 0;
    Plan P;
    int rc = make_plan(P, batch, H, W, C, C, r, eps, s, sub_mode);
    if (rc) return rc;
    if (!std::isfinite(gain) || gain < 0.0) return FGF_ERR_PARAM;
    if ((rc = check_pointers(I, I, out, P, true))) return rc;
    // out = (I - q) gain + q = gain I + (1 - gain)(mean_a^T I + mean_b): fold into the maps
    P.k1 = (float)(1.0 - gain);
    P.k0 = (float)gain;
    return run_all(I, I, out, P, workspace, ws_bytes, static_cast<cudaStream_t>(cuda_stream));
}

size_t fgf_enhance_workspace_bytes(int batch, int H, int W, int C, int r, int s, int guide) {
    if (guide == FGF_GUIDE_LUMA && C == 3) {
        // [luminance planes][the workspace of the gray-guided filter with 3 input channels]
        Plan P0, P1;
        if (make_plan(P0, batch, H, W, 1, 3, r, 1.0, s, FGF_SUB_NEAREST) ||
            make_plan(P1, batch, H, W, 1, 3, r, 1.0, s, FGF_SUB_BILINEAR))
            return 0;
        return align_up((size_t)batch * H * W * sizeof(float)) +
               std::max(plan_ws(P0, true), plan_ws(P1, true));
    }
    if (guide != FGF_GUIDE_SELF && guide != FGF_GUIDE_LUMA) return 0;
    return fgf_workspace_bytes(batch, H, W, C, C, r, s);
}

int fgf_enhance_ex_ws(const float* I, float* out, int batch, int H, int W, int C, int r,
                      double eps, int s, int sub_mode, double gain, int guide, void* workspace,
                      size_t ws_bytes, void* cuda_stream) {
    if (guide != FGF_GUIDE_SELF && guide != FGF_GUIDE_LUMA) return FGF_ERR_PARAM;
    if (guide == FGF_GUIDE_SELF || C == 1)
        return fgf_enhance_ws(I, out, batch, H, W, C, r, eps, s, sub_mode, gain, workspace,
                              ws_bytes, cuda_stream);
    g_last_launches = 0;
    Plan P;   // SPEC's shared gray guidance: I = to_grayscale(img), p = img (3 channels)
    int rc = make_plan(P, batch, H, W, 1, 3, r, eps, s, sub_mode);
    if (rc) return rc;
    if (!std::isfinite(gain) || gain < 0.0) return FGF_ERR_PARAM;
    if (!I || !out || !workspace) return FGF_ERR_NULL;
    if ((reinterpret_cast<uintptr_t>(I) | reinterpret_cast<uintptr_t>(out)) & 3u) return FGF_ERR_ALIGN;
    const size_t img_bytes = (size_t)batch * 3 * P.N * sizeof(float);
    if (overlaps(out, img_bytes, I, img_bytes)) return FGF_ERR_ALIAS;
    if (!is_device_ptr(I) || !is_device_ptr(out) || !is_device_ptr(workspace)) return FGF_ERR_DEVICE;
    const size_t o_lw = align_up((size_t)batch * P.N * sizeof(float));
    if (ws_bytes < o_lw + plan_ws(P, true)) return FGF_ERR_NOMEM;
    cudaStream_t st = static_cast<cudaStream_t>(cuda_stream);
    float* L = static_cast<float*>(workspace);
    if ((rc = launch_luma(I, L, batch, P.N, st))) return rc;
    int launches = g_last_launches;
    g_last_launches = 0;
    if ((rc = run_all(L, I, out, P, static_cast<char*>(workspace) + o_lw, ws_bytes - o_lw, st)))
        return rc;
    launches += g_last_launches;
    g_last_launches = 0;
    rc = launch_blend(I, out, (size_t)batch * 3 * P.N, gain, st);
    g_last_launches += launches;
    return rc;
}

int fgf_filter(const float* I, const float* p, float* q, int batch, int H, int W, int C_I,
               int C_p, int r, double eps, int s, int sub_mode) {
    g_last_launches = 0;
    Plan P;
    int rc = make_plan(P, batch, H, W, C_I, C_p, r, eps, s, sub_mode);
    if (rc) return rc;
    if ((rc = check_pointers(I, p, q, P, true))) return rc;
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return FGF_ERR_CUDA;
    const size_t need = plan_ws(P, true);
    std::lock_guard<std::mutex> lk(g_ws_mu);
    if ((int)g_ws.size() <= dev) g_ws.resize(dev + 1);
    DevWs& d = g_ws[dev];
    if (d.bytes < need) {
        if (d.ptr) {
            cudaDeviceSynchronize();
            cudaFree(d.ptr);
            d.ptr = nullptr;
            d.bytes = 0;
        }
        if (cudaMalloc(&d.ptr, need) != cudaSuccess) {
            cudaGetLastError();
            return FGF_ERR_NOMEM;
        }
        d.bytes = need;
    }
    return run_all(I, p, q, P, d.ptr, d.bytes, nullptr);
}

int fgf_coefficients(const float* I, const float* p, float* mean_ab, int batch, int H, int W,
                     int C_I, int C_p, int r, double eps, int s, int sub_mode, void* workspace,
                     size_t ws_bytes, void* cuda_stream) {
    g_last_launches = 0;
    Plan P;
    int rc = make_plan(P, batch, H, W, C_I, C_p, r, eps, s, sub_mode);
    if (rc) return rc;
    if (!I || !p || !mean_ab) return FGF_ERR_NULL;
    if ((reinterpret_cast<uintptr_t>(I) | reinterpret_cast<uintptr_t>(p) |
         reinterpret_cast<uintptr_t>(mean_ab)) & 3u)
        return FGF_ERR_ALIGN;
    if (!is_device_ptr(I) || !is_device_ptr(p) || !is_device_ptr(mean_ab)) return FGF_ERR_DEVICE;
    return run_coefficients(I, p, mean_ab, P, workspace, ws_bytes,
                            static_cast<cudaStream_t>(cuda_stream));
}

int fgf_upsample_output(const float* I, const float* mean_ab, float* q, int batch, int H, int W,
                        int C_I, int C_p, int s, void* cuda_stream) {
    g_last_launches = 0;
    Plan P;
    int rc = make_plan(P, batch, H, W, C_I, C_p, 1, 1.0, s, FGF_SUB_NEAREST);
    if (rc) return rc;
    if (!I || !mean_ab || !q) return FGF_ERR_NULL;
    if ((reinterpret_cast<uintptr_t>(I) | reinterpret_cast<uintptr_t>(mean_ab) |
         reinterpret_cast<uintptr_t>(q)) & 3u)
        return FGF_ERR_ALIGN;
    const size_t bq = (size_t)batch * C_p * P.N * 4;
    if (overlaps(q, bq, I, (size_t)batch * C_I * P.N * 4) ||
        overlaps(q, bq, mean_ab, (size_t)batch * P.NC * P.n * 4))
        return FGF_ERR_ALIAS;
    if (!is_device_ptr(I) || !is_device_ptr(mean_ab) || !is_device_ptr(q)) return FGF_ERR_DEVICE;
    return launch_output(I, mean_ab, q, batch, P, static_cast<cudaStream_t>(cuda_stream));
}

int fgf_subsample(const float* src, float* dst, int planes, int H, int W, int s, int sub_mode,
                  void* cuda_stream) {
    g_last_launches = 0;
    if (planes < 1 || H < 1 || W < 1) return FGF_ERR_SHAPE;
    if (s < 1 || (sub_mode != FGF_SUB_NEAREST && sub_mode != FGF_SUB_BILINEAR)) return FGF_ERR_PARAM;
    if (!src || !dst) return FGF_ERR_NULL;
    if ((reinterpret_cast<uintptr_t>(src) | reinterpret_cast<uintptr_t>(dst)) & 3u) return FGF_ERR_ALIGN;
    if (!is_device_ptr(src) || !is_device_ptr(dst)) return FGF_ERR_DEVICE;
    const size_t N = (size_t)H * W;
    const size_t n = (size_t)lowres_dim(H, s) * lowres_dim(W, s);
    if (overlaps(dst, (size_t)planes * n * 4, src, (size_t)planes * N * 4)) return FGF_ERR_ALIAS;
    if (N >= (1ull << 31)) return FGF_ERR_UNSUPPORTED;
    cudaStream_t st = static_cast<cudaStream_t>(cuda_stream);
    if (s == 1) {
        if (cudaMemcpyAsync(dst, src, (size_t)planes * N * 4, cudaMemcpyDeviceToDevice, st))
            return FGF_ERR_CUDA;
        return FGF_OK;
    }
    Plan P{};
    P.H = H; P.W = W; P.s = s; P.sub = sub_mode;
    P.h = lowres_dim(H, s); P.w = lowres_dim(W, s);
    return launch_subsample(src, dst, planes, P, st);
}

size_t fgf_lowres_workspace_bytes(int batch, int h, int w, int C_I, int C_p) {
    // radius-independent: enough for every engine the low-res chain may take (K13 needs none;
    // the strip engine its a, b maps; K5 its hb rings, largest over the radii it serves)
    Plan P;
    if (make_plan(P, batch, h, w, C_I, C_p, 1, 1.0, 1, FGF_SUB_NEAREST)) return 0;
    const size_t chunk = (size_t)std::max(1, std::min(batch, (int)std::max<size_t>(
        1, kChunkTargetBytes / std::max<size_t>(1, (size_t)2 * P.NC * P.n * sizeof(float)))));
    size_t ring = 0;
    if (C_I == 1)
        for (int R = 2; 4 * R + 32 <= kWideMaxCols; ++R) ring = std::max(ring, wide_ring_reserve(R, C_p));
    return std::max<size_t>(kAlign, align_up(chunk * P.NC * P.n * sizeof(float)) + ring);
}

int fgf_lowres_mean(const float* Is, const float* ps, float* mean_ab, int batch, int h, int w,
                    int C_I, int C_p, int r_low, double eps, void* workspace, size_t ws_bytes,
                    void* cuda_stream) {
    // Steps 2-5 on given low-res planes: exactly the s = 1 path with radius r'.
    return fgf_coefficients(Is, ps, mean_ab, batch, h, w, C_I, C_p, r_low, eps, 1,
                            FGF_SUB_NEAREST, workspace, ws_bytes, cuda_stream);
}

int fgf_upsample_output_rows(const float* I, const float* mean_ab, float* q, int batch, int rows,
                             int W, int C_I, int C_p, int H_total, int h_total, int w, int Y0,
                             int y0_maps, int h_maps, void* cuda_stream) {
    g_last_launches = 0;
    if (batch < 1 || rows < 1 || W < 1 || w < 1 || w > W || H_total < 1 || h_total < 1 ||
        h_total > H_total || h_maps < 1)
        return FGF_ERR_SHAPE;
    if ((C_I != 1 && C_I != 3) || C_p < 1 || C_p > 4) return FGF_ERR_SHAPE;
    if (Y0 < 0 || Y0 + rows > H_total || y0_maps < 0 || y0_maps + h_maps > h_total)
        return FGF_ERR_PARAM;
    // The rows' low-res sources (R5, global map) must lie inside the maps buffer.
    auto src_lo = [&](int Y) {
        long long num = (long long)(2 * Y + 1) * h_total - H_total;
        if (num <= 0) return 0;
        return (int)std::min<long long>(num / (2LL * H_total), h_total - 1);
    };
    if (src_lo(Y0) < y0_maps || std::min(src_lo(Y0 + rows - 1) + 1, h_total - 1) >= y0_maps + h_maps)
        return FGF_ERR_PARAM;
    if (!I || !mean_ab || !q) return FGF_ERR_NULL;
    if ((reinterpret_cast<uintptr_t>(I) | reinterpret_cast<uintptr_t>(mean_ab) |
         reinterpret_cast<uintptr_t>(q)) & 3u)
        return FGF_ERR_ALIGN;
    const int NC = (C_I + 1) * C_p;
    const size_t N = (size_t)rows * W, n = (size_t)h_maps * w;
    if (N * std::max(C_I, C_p) >= (1ull << 31) || n * NC >= (1ull << 31)) return FGF_ERR_UNSUPPORTED;
    const size_t bq = (size_t)batch * C_p * N * 4;
    if (overlaps(q, bq, I, (size_t)batch * C_I * N * 4) ||
        overlaps(q, bq, mean_ab, (size_t)batch * NC * n * 4))
        return FGF_ERR_ALIAS;
    if (!is_device_ptr(I) || !is_device_ptr(mean_ab) || !is_device_ptr(q)) return FGF_ERR_DEVICE;
    Plan P{};
    P.batch = batch; P.H = rows; P.W = W; P.CI = C_I; P.CP = C_p; P.NC = NC;
    P.h = h_maps; P.w = w; P.N = N; P.n = n; P.TR = 32;
    const Band band{H_total, h_total, Y0, y0_maps, h_maps};
    return launch_output(I, mean_ab, q, batch, P, static_cast<cudaStream_t>(cuda_stream), &band);
}

// fgf_filter_host copies only the sample rows of p when the subsampling is nearest (s > 1) and
// the rows are long enough (>= 2 KB) for the copy engine's 2-D transfers to run at link rate.
static bool host_p_sample_rows(const Plan& P) {
    return P.s > 1 && P.sub == FGF_SUB_NEAREST && (size_t)P.W * P.esize >= 2048;
}

size_t fgf_filter_host_input_bytes(int batch, int H, int W, int C_I, int C_p, int r, int s,
                                   int sub_mode, int dtype, int self_guided) {
    Plan P;
    if (make_plan(P, batch, H, W, C_I, C_p, r, 0.01, s, sub_mode) || set_dtype(P, dtype)) return 0;
    const bool self = self_guided && C_I == 1 && C_p == 1;
    size_t b = (size_t)batch * C_I * P.N * P.esize;
    if (!self)
        b += (size_t)batch * C_p * P.esize * (host_p_sample_rows(P) ? (size_t)P.h * P.W : P.N);
    return b;
}

int fgf_filter_host_ex(const void* I, const void* p, void* q, int batch, int H, int W, int C_I,
                       int C_p, int r, double eps, int s, int sub_mode, int dtype, int device) {
    g_last_launches = 0;
    Plan P;
    int rc = make_plan(P, batch, H, W, C_I, C_p, r, eps, s, sub_mode);
    if (rc) return rc;
    if ((rc = set_dtype(P, dtype))) return rc;
    if (dtype != FGF_F32 && !(C_I * 10 + C_p == 11 || C_I * 10 + C_p == 31 || C_I * 10 + C_p == 33))
        return FGF_ERR_UNSUPPORTED;
    if ((rc = check_pointers(I, p, q, P, false))) return rc;
    if (cudaSetDevice(device) != cudaSuccess) return FGF_ERR_CUDA;
    const bool self = (I == p) && C_I == 1 && C_p == 1;
    const size_t es = P.esize;
    const char* Ih = static_cast<const char*>(I);
    const char* ph = static_cast<const char*>(p);
    char* qh = static_cast<char*>(q);

    // Sub-batch per pipeline slot: ~256 MB of I+p+q, at least one image; the I, p and q parts
    // of a slot start on 256-byte boundaries.
    const size_t img_bytes = (size_t)(C_I + (self ? 0 : C_p) + C_p) * P.N * es;
    // ... and at least four chunks when the batch has four images, so that a small batch still
    // overlaps its copies with the filter (the development knob sets the slot size alone).
    size_t slot_target = 256u << 20;
    int sb_cap = std::max(1, (batch + 3) / 4);
    if (const char* e = dev_env("FGF_HOST_CHUNK_MB")) {
        slot_target = (size_t)std::max(1, atoi(e)) << 20;
        sb_cap = batch;
    }
    const int sb = (int)std::max<size_t>(
        1, std::min<size_t>(std::min(batch, sb_cap), slot_target / img_bytes));
    Plan Psub;
    make_plan(Psub, sb, H, W, C_I, C_p, r, eps, s, sub_mode);
    set_dtype(Psub, dtype);
    const size_t partI = align_up((size_t)sb * C_I * P.N * es);
    const size_t partP = self ? 0 : align_up((size_t)sb * C_p * P.N * es);
    const size_t slot_bytes = partI + partP + align_up((size_t)sb * C_p * P.N * es);
    const size_t need_ws = plan_ws(Psub, true);

    std::lock_guard<std::mutex> lk(g_host_mu);
    if ((int)g_host.size() <= device) g_host.resize(device + 1);
    HostPipe& hp = g_host[device];
    if (!hp.init) {
        if (cudaStreamCreateWithFlags(&hp.s_h2d, cudaStreamNonBlocking) ||
            cudaStreamCreateWithFlags(&hp.s_comp, cudaStreamNonBlocking) ||
            cudaStreamCreateWithFlags(&hp.s_d2h, cudaStreamNonBlocking))
            return FGF_ERR_CUDA;
        for (int k = 0; k < 2; ++k) {
            if (cudaEventCreateWithFlags(&hp.ev_in[k], cudaEventDisableTiming) ||
                cudaEventCreateWithFlags(&hp.ev_done[k], cudaEventDisableTiming) ||
                cudaEventCreateWithFlags(&hp.ev_free[k], cudaEventDisableTiming))
                return FGF_ERR_CUDA;
        }
        for (int k = 0; k < kHostBands; ++k)
            if (cudaEventCreateWithFlags(&hp.ev_bin[k], cudaEventDisableTiming) ||
                cudaEventCreateWithFlags(&hp.ev_bout[k], cudaEventDisableTiming))
                return FGF_ERR_CUDA;
        hp.init = true;
    }
    if (hp.dbytes < slot_bytes) {
        cudaDeviceSynchronize();
        for (int k = 0; k < 2; ++k) {
            if (hp.dbuf[k]) cudaFree(hp.dbuf[k]);
            hp.dbuf[k] = nullptr;
        }
        hp.dbytes = 0;
        for (int k = 0; k < 2; ++k)
            if (cudaMalloc(&hp.dbuf[k], slot_bytes) != cudaSuccess) {
                cudaGetLastError();
                return FGF_ERR_NOMEM;
            }
        hp.dbytes = slot_bytes;
    }
    if (hp.wsbytes < need_ws) {
        cudaDeviceSynchronize();
        if (hp.ws) cudaFree(hp.ws);
        hp.ws = nullptr;
        hp.wsbytes = 0;
        if (cudaMalloc(&hp.ws, need_ws) != cudaSuccess) {
            cudaGetLastError();
            return FGF_ERR_NOMEM;
        }
        hp.wsbytes = need_ws;
    }

    // Once a copy is enqueued the caller's host buffers are in use: every return below
    // drains the three streams first, so no copy still reads I / p or writes q afterwards.
    auto drain = [&](int status) {
        const bool ok = cudaStreamSynchronize(hp.s_h2d) == cudaSuccess &&
                        cudaStreamSynchronize(hp.s_comp) == cudaSuccess &&
                        cudaStreamSynchronize(hp.s_d2h) == cudaSuccess;
        if (!ok) cudaGetLastError();
        return status != FGF_OK ? status : (ok ? FGF_OK : FGF_ERR_CUDA);
    };
    int launches = 0;
    // ONE gray frame (any element type), nearest samples: whole-image chunks cannot overlap anything, so the
    // frame is pipelined by rows instead.  The sample rows of I and p go first and the low-res
    // chain (steps 1-5) runs on them while the other rows of I follow in kHostBands bands; each
    // band's output pass (steps 6-7, global vertical map) starts when its rows have arrived
    // and its q rows leave while the next band is still coming in.
    const bool frame_bands = batch == 1 && C_I == 1 && C_p == 1 &&
                             host_p_sample_rows(P) && !P.fused_out && P.h >= 4 * kHostBands &&
                             dev_env("FGF_HOST_NOBANDS") == nullptr;
    if (frame_bands) {
        char* dI = reinterpret_cast<char*>(hp.dbuf[0]);
        char* dp = self ? dI : dI + partI;
        char* dq = dI + partI + partP;
        const size_t rowb = (size_t)W * es, pitch = (size_t)s * rowb;
        if (cudaMemcpy2DAsync(dI, pitch, Ih, pitch, rowb, P.h, cudaMemcpyHostToDevice, hp.s_h2d))
            return drain(FGF_ERR_CUDA);
        if (!self && cudaMemcpy2DAsync(dp, pitch, ph, pitch, rowb, P.h, cudaMemcpyHostToDevice, hp.s_h2d))
            return drain(FGF_ERR_CUDA);
        if (cudaEventRecord(hp.ev_in[0], hp.s_h2d) || cudaStreamWaitEvent(hp.s_comp, hp.ev_in[0], 0))
            return drain(FGF_ERR_CUDA);
        float* mean = reinterpret_cast<float*>(static_cast<char*>(hp.ws) + mean_off(P));
        if ((rc = run_lowres(dI, dp, mean, 0, 1, P, static_cast<char*>(hp.ws), hp.s_comp)))
            return drain(rc);
        launches += g_last_launches;
        g_last_launches = 0;
        const int hb = (P.h + kHostBands - 1) / kHostBands;   // low-res rows per band
        for (int k = 0; k * hb < P.h; ++k) {
            const int Y0 = k * hb * s, Y1 = std::min(H, (k + 1) * hb * s), rows = Y1 - Y0;
            // rows y s + 1 .. y s + s - 1 of the band's full groups, then a partial last group
            const int groups = rows / s, rem = rows - groups * s;
            const size_t o = (size_t)Y0 * rowb;
            if (groups > 0 && cudaMemcpy2DAsync(dI + o + rowb, pitch, Ih + o + rowb, pitch,
                                                (size_t)(s - 1) * rowb, groups,
                                                cudaMemcpyHostToDevice, hp.s_h2d))
                return drain(FGF_ERR_CUDA);
            if (rem > 1 && cudaMemcpyAsync(dI + o + (size_t)groups * pitch + rowb,
                                           Ih + o + (size_t)groups * pitch + rowb,
                                           (size_t)(rem - 1) * rowb, cudaMemcpyHostToDevice, hp.s_h2d))
                return drain(FGF_ERR_CUDA);
            if (cudaEventRecord(hp.ev_bin[k], hp.s_h2d) ||
                cudaStreamWaitEvent(hp.s_comp, hp.ev_bin[k], 0))
                return drain(FGF_ERR_CUDA);
            Plan Pr{};
            Pr.batch = 1; Pr.H = rows; Pr.W = W; Pr.CI = 1; Pr.CP = 1; Pr.NC = P.NC;
            Pr.h = P.h; Pr.w = P.w; Pr.N = (size_t)rows * W; Pr.n = P.n; Pr.TR = 32;
            Pr.s = s; Pr.sub = sub_mode; Pr.r = r; Pr.R = P.R; Pr.eps = eps;
            Pr.dtype = dtype; Pr.esize = (int)es;
            const Band band{H, P.h, Y0, 0, P.h};
            if ((rc = launch_output(dI + o, mean, dq + o, 1, Pr, hp.s_comp, &band))) return drain(rc);
            launches += g_last_launches;
            g_last_launches = 0;
            if (cudaEventRecord(hp.ev_bout[k], hp.s_comp) ||
                cudaStreamWaitEvent(hp.s_d2h, hp.ev_bout[k], 0))
                return drain(FGF_ERR_CUDA);
            if (cudaMemcpyAsync(qh + o, dq + o, (size_t)rows * rowb, cudaMemcpyDeviceToHost, hp.s_d2h))
                return drain(FGF_ERR_CUDA);
        }
        if ((rc = drain(FGF_OK))) return rc;
        g_last_launches = launches;
        return FGF_OK;
    }
    int k = 0;
    for (int b0 = 0; b0 < batch; b0 += sb, ++k) {
        const int nb = std::min(sb, batch - b0);
        const int slot = k & 1;
        char* dI = reinterpret_cast<char*>(hp.dbuf[slot]);
        char* dp = self ? dI : dI + partI;
        char* dq = dI + partI + partP;
        // The slot is free once the D2H of chunk k-2 has finished.
        if (k >= 2 && cudaStreamWaitEvent(hp.s_h2d, hp.ev_free[slot], 0)) return drain(FGF_ERR_CUDA);
        if (cudaMemcpyAsync(dI, Ih + (size_t)b0 * C_I * P.N * es, (size_t)nb * C_I * P.N * es,
                            cudaMemcpyHostToDevice, hp.s_h2d))
            return drain(FGF_ERR_CUDA);
        if (!self && !host_p_sample_rows(P)) {
            if (cudaMemcpyAsync(dp, ph + (size_t)b0 * C_p * P.N * es, (size_t)nb * C_p * P.N * es,
                                cudaMemcpyHostToDevice, hp.s_h2d))
                return drain(FGF_ERR_CUDA);
        } else if (!self) {
            // Nearest samples (R3): Alg. 2 reads p only at p[y s][x s] (q = mean_a I +
            // mean_b needs I alone at full resolution), and every engine addresses p
            // through the row stride s W -- only rows y s cross the host link.  The device
            // plane keeps its full geometry; its other rows are never read.
            const size_t pitch = (size_t)s * W * es, width = (size_t)W * es;
            const char* pc = ph + (size_t)b0 * C_p * P.N * es;
            if (H % s == 0) {   // one pitch across the chunk's planes
                if (cudaMemcpy2DAsync(dp, pitch, pc, pitch, width, (size_t)nb * C_p * P.h,
                                      cudaMemcpyHostToDevice, hp.s_h2d))
                    return drain(FGF_ERR_CUDA);
            } else {
                for (int j = 0; j < nb * C_p; ++j)
                    if (cudaMemcpy2DAsync(dp + (size_t)j * P.N * es, pitch, pc + (size_t)j * P.N * es,
                                          pitch, width, P.h, cudaMemcpyHostToDevice, hp.s_h2d))
                        return drain(FGF_ERR_CUDA);
            }
        }
        if (cudaEventRecord(hp.ev_in[slot], hp.s_h2d) ||
            cudaStreamWaitEvent(hp.s_comp, hp.ev_in[slot], 0))
            return drain(FGF_ERR_CUDA);
        Plan Pc;
        if ((rc = make_plan(Pc, nb, H, W, C_I, C_p, r, eps, s, sub_mode))) return drain(rc);
        if ((rc = set_dtype(Pc, dtype))) return drain(rc);
        if ((rc = run_all(dI, dp, dq, Pc, hp.ws, hp.wsbytes, hp.s_comp))) return drain(rc);
        launches += g_last_launches;
        g_last_launches = 0;
        if (cudaEventRecord(hp.ev_done[slot], hp.s_comp) ||
            cudaStreamWaitEvent(hp.s_d2h, hp.ev_done[slot], 0))
            return drain(FGF_ERR_CUDA);
        if (cudaMemcpyAsync(qh + (size_t)b0 * C_p * P.N * es, dq, (size_t)nb * C_p * P.N * es,
                            cudaMemcpyDeviceToHost, hp.s_d2h))
            return drain(FGF_ERR_CUDA);
        if (cudaEventRecord(hp.ev_free[slot], hp.s_d2h)) return drain(FGF_ERR_CUDA);
    }
    if ((rc = drain(FGF_OK))) return rc;
    g_last_launches = launches;
    return FGF_OK;
}

int fgf_filter_host(const float* I, const float* p, float* q, int batch, int H, int W, int C_I,
                    int C_p, int r, double eps, int s, int sub_mode, int device) {
    return fgf_filter_host_ex(I, p, q, batch, H, W, C_I, C_p, r, eps, s, sub_mode, FGF_F32, device);
}

}  // extern "C"
