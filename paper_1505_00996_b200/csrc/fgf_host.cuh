// fgf_host.cuh -- internal host-side declarations shared by the translation units of
// libfgf.so: the launch plan, per-launch profiling / NVTX scopes, launch helpers and the
// launcher entry points of each kernel family.  Each family is its own translation unit
// (fgf_k_stats.cu, fgf_k_mean.cu, fgf_k_out.cu, fgf_k_lowres.cu) so that the build compiles
// them in parallel, each in one ptxas pass (deterministic register allocation).
#pragma once
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <vector>

#include <nvtx3/nvToolsExt.h>   // header-only NVTX v3: ranges cost ~nothing without a tool

#include "../../include/fgf.h"
#include "fgf_kernels.cuh"
#include "fgf_lowres.cuh"
#include "fgf_wide.cuh"

namespace fgf {

extern thread_local int g_last_launches;   // launches of the last API call (fgf_api.cu)

constexpr size_t kAlign = 256;
constexpr size_t kChunkTargetBytes = 8ull << 30;  // low-res workspace bytes per pipeline slot

// ---- optional per-launch event timing (fgf_profile_*)
enum { KIND_SUB = 0, KIND_STATS = 1, KIND_MEAN = 2, KIND_OUT = 3, KIND_LOWRES = 4, KIND_WIDE = 5,
       KIND_TINY = 6, NKIND = 7 };
struct ProfRec {
    int kind;
    cudaEvent_t a, b;
};
struct Profiler {
    bool on = false;
    std::vector<ProfRec> recs;
    std::vector<cudaEvent_t> pool;
    cudaEvent_t get() {
        if (!pool.empty()) {
            cudaEvent_t e = pool.back();
            pool.pop_back();
            return e;
        }
        cudaEvent_t e = nullptr;
        cudaEventCreate(&e);
        return e;
    }
    void clear() {
        for (auto& r : recs) {
            pool.push_back(r.a);
            pool.push_back(r.b);
        }
        recs.clear();
    }
};
extern Profiler g_prof;                   // fgf_api.cu

const char* const kKindName[NKIND] = {"fgf K0 subsample", "fgf K1 statistics+coefficients",
                                      "fgf K3 box of a,b", "fgf K4 upsample+output",
                                      "fgf K13 fused low-res chain",
                                      "fgf K5 radius-independent fused chain",
                                      "fgf K6 single-kernel small image"};

// Around every launch: an NVTX range named after the kernel (timeline tools: nsys, ncu
// --nvtx) and, when fgf_profile_enable(1) is on, a CUDA-event pair on the launching stream.
struct ProfScope {
    cudaStream_t st;
    int kind;
    cudaEvent_t a = nullptr;
    ProfScope(int k, cudaStream_t s) : st(s), kind(k) {
        nvtxRangePushA(kKindName[k]);
        if (g_prof.on) {
            a = g_prof.get();
            cudaEventRecord(a, st);
        }
    }
    ~ProfScope() {
        if (a) {
            cudaEvent_t b = g_prof.get();
            cudaEventRecord(b, st);
            g_prof.recs.push_back({kind, a, b});
        }
        nvtxRangePop();
    }
};

inline size_t align_up(size_t x) { return (x + kAlign - 1) / kAlign * kAlign; }

// Engine of steps 2-5 (and, for K5 at s = 1, of the whole filter), chosen once per plan.
enum { ENG_STRIP = 0, ENG_K13 = 1, ENG_WIDE = 2, ENG_TINY = 3 };

// K5 geometry (fgf_k_wide.cu): strips of TW output columns, segments of TH rows, a persistent
// grid of `grid` CTAs of NT threads, one hb ring of ring_bytes / grid per CTA.
struct WideGeom {
    int TW = 0, NT = 0, strips = 0, segs = 0, TH = 0, items = 0, grid = 0, R = 0;
    size_t ring_bytes = 0;
};

struct Plan {
    int batch, H, W, CI, CP, r, s, sub;
    double eps;
    float k1 = 1.0f, k0 = 0.0f;   // mean-map fold (detail enhancement), identity by default
    int dtype = FGF_F32;          // element type of I, p, q (FGF_F32 / FGF_F16 / FGF_BF16)
    int esize = 4;                // its bytes
    int h, w, R, NC;
    size_t N, n;
    int chunk;
    // strip box engine
    int nt, TW, strips;
    // output kernel
    int TR;
    // engine and workspace carve-up per pipeline slot (bytes), from plan_layout()
    int engine = ENG_STRIP;
    bool fused_out = false;       // K5 at s = 1: one kernel writes q (no mean maps, no K4)
    bool pdl_out = false;         // K4 launched as a programmatic dependent of K13 (run_all)
    size_t ws_planes, ws_coef, ws_mean, ws_ring, ws_slot;
    int nslots;
};

// --------------------------------------------------------------------- launch helpers

template <typename K>
void set_smem(K kernel, size_t bytes) {
    if (bytes > 48 * 1024)
        cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
}

// Development knobs: environment variables that select another CUDA kernel
// variant or geometry of the same computation, for tests and sweeps.  The library honours
// them only when FGF_DEV=1 is set too, so a caller's stray environment cannot change which
// kernels a call runs.
inline const char* dev_env(const char* name) {
    const char* d = getenv("FGF_DEV");
    if (!d || atoi(d) == 0) return nullptr;
    return getenv(name);
}

// FGF_DEBUG_SYNC=1: synchronise after every launch so that an asynchronous fault is reported
// by the call (and the kernel) that caused it, not at the caller's next synchronisation.
inline bool debug_sync() {
    const char* e = getenv("FGF_DEBUG_SYNC");   // read per launch: a few per call
    return e && atoi(e) != 0;
}

inline int last_error() {
    if (cudaGetLastError() != cudaSuccess) return FGF_ERR_CUDA;
    if (debug_sync() && cudaDeviceSynchronize() != cudaSuccess) return FGF_ERR_CUDA;
    return FGF_OK;
}

// Row band of a taller image: I/q hold rows [Yoff, Yoff + P.H) of an image of height Hg;
// the maps buffer holds low-res rows [yoff, yoff + hm) of a low-res image of height hg.
struct Band {
    int Hg, hg, Yoff, yoff, hm;
};

// ---- launcher entry points (each returns an FGF_* status; launches go on stream st)
// K0 (fgf_k_mean.cu): step 1 into compact fp32 low-res planes.
int launch_subsample(const void* src, float* dst, int planes, const Plan& P, cudaStream_t st);
// ... planes from src then planes2 from src2 in one launch, into consecutive dst planes
int launch_subsample2(const void* src, int planes, const void* src2, int planes2, float* dst,
                      const Plan& P, cudaStream_t st);
// K1 / K3 strip engine (fgf_k_stats.cu: MODE_STATS, fgf_k_mean.cu: MODE_MEAN).
template <int MODE>
int launch_strip(const StripParams& sp, int images, const Plan& P, cudaStream_t st);
extern template int launch_strip<MODE_STATS>(const StripParams&, int, const Plan&, cudaStream_t);
extern template int launch_strip<MODE_MEAN>(const StripParams&, int, const Plan&, cudaStream_t);
// K4 (fgf_k_out.cu); band: a row band of a taller image (nullptr: whole images).
int launch_output(const void* I, const float* M, void* q, int images, const Plan& P,
                  cudaStream_t st, const Band* band = nullptr);
int lowres_span(int T, int n_dst, int n_src);
// K5 (fgf_k_wide.cu): geometry for `images` images, and the launch (maps or, outq, q).
bool wide_geom(WideGeom& g, int h, int w, int R, int CP, int images, bool outq);
bool wide_supports(int CP, int dtype);
size_t wide_ring_reserve(int R, int CP);
int launch_wide(const WideParams& wp, const WideGeom& g, int CP, int dtype, bool outq,
                cudaStream_t st);
// Application kernels (fgf_k_apps.cu): SPEC to_grayscale, and out = gain img + (1 - gain) q.
int launch_luma(const float* img, float* L, int batch, size_t N, cudaStream_t st);
int launch_blend(const float* img, float* q, size_t n, double gain, cudaStream_t st);
// K6 (fgf_k_tiny.cu): the whole filter of small gray images in one kernel.
bool tiny_supports(const Plan& P);
int launch_tiny(const float* I, const float* p, float* q, const Plan& P, cudaStream_t st);
// K13 (fgf_k_lowres.cu); dry = true: only report whether K13 serves this plan.
int launch_lowres_gray(const LowresParams& lp, int images, const Plan& P, cudaStream_t st,
                       bool dry = false);

}  // namespace fgf
