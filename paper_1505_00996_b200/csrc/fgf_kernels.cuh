// fgf_kernels.cuh -- sm_100a kernels of the Fast Guided Filter hot path.
//
// Algorithm 2 of He & Sun, "Fast Guided Filter", as four kernels:
//
//   K0 subsample_block_kernel  step 1 for "bilinear" (= clipped s x s block mean,
//                         DESIGN.md R4) subsampling only: I', p' into compact low-res planes.
//                         Nearest subsampling (R3) needs no pass: K1 reads the sample sites
//                         I[y*s][x*s] straight from the full-resolution image.
//   K1 box_strip_kernel<STATS>  steps 1-4 (Eq.2-3): the 4 (gray) / 9+4C_p (color)
//                         box means of I', p', I'I'^T, I'p'^T, then the coefficient epilogue
//                         a, b (gray closed form, color 3x3 symmetric adjugate), all fp64.
//   K3 box_strip_kernel<MEAN>   step 5: mean_a, mean_b = f_mean(a, b), fp64 sums.
//   K4 output_kernel      steps 6-7: bilinear upsample of mean_a, mean_b and
//                         q = mean_a^T I + mean_b with the FULL-resolution I.
//
// Box engine (K1/K3).  A CTA owns a strip of TW low-res output columns and a segment of TH
// output rows; it reads the halo columns [x0-R, x0+TW+R) clipped to the image.  One thread
// per halo column keeps fp64 running sums of every statistic map in registers while it walks
// down the rows (add row y+R, subtract row y-R-1: O(1) per row, "independent of the
// filter size").  Every G rows the column sums are snapshot to shared memory and each warp
// slides a horizontal window along one row in runs of K (odd) columns, so the 16 lanes of a
// half-warp hit 16 distinct fp64 banks.  The next G rows' loads are issued before the
// horizontal phase (software pipelining) and results are staged in shared memory so the
// global stores are coalesced.  Borders: clip-and-renormalize, counts are in-bounds counts
// (R1).
//
// Nothing here is shared with oracle/ (the independent CPU reference).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace fgf {

enum { MODE_STATS = 0, MODE_MEAN = 1 };

// ------------------------------------------------------------------ K0: block-mean subsample

struct SubParams {
    const float* src;       // [plane][H][W]
    float* dst;             // [plane][h][w]
    int H, W, h, w, s;
    int rows_per_cta;       // low-res rows per CTA (grid-y covers h / rows_per_cta)
};

// R4: mean of the clipped s x s block, summed in fp64.  One thread per
// low-res column, several low-res rows per CTA for memory-level parallelism.
// grid (ceil(w/256), ceil(h/rows_per_cta), planes).
template <bool VEC4>
__global__ void __launch_bounds__(256) subsample_block_kernel(SubParams P) {
    const int x = blockIdx.x * blockDim.x + threadIdx.x;
    if (x >= P.w) return;
    const size_t plane = blockIdx.z;
    const float* src = P.src + plane * (size_t)P.H * P.W;
    float* dst = P.dst + plane * (size_t)P.h * P.w;
    const int y0 = blockIdx.y * P.rows_per_cta;
    const int y1 = min(P.h, y0 + P.rows_per_cta);
    const int xa = x * P.s, xb = min(P.W, xa + P.s);
    for (int y = y0; y < y1; ++y) {
        const int ya = y * P.s, yb = min(P.H, ya + P.s);
        double acc = 0.0;
        if (VEC4) {  // s == 4, W % 4 == 0, 16-byte aligned rows
            for (int yy = ya; yy < yb; ++yy) {
                const float4 v = __ldcs(reinterpret_cast<const float4*>(src + (size_t)yy * P.W) + x);
                acc += (double)v.x;
                acc += (double)v.y;
                acc += (double)v.z;
                acc += (double)v.w;
            }
        } else {
            for (int yy = ya; yy < yb; ++yy) {
                const float* row = src + (size_t)yy * P.W;
                for (int xx = xa; xx < xb; ++xx) acc += (double)__ldcs(row + xx);
            }
        }
        dst[(size_t)y * P.w + x] = (float)(acc / (double)((yb - ya) * (xb - xa)));
    }
}

// R3: nearest = top-left sample I[y*s][x*s], compacted into low-res planes so
// that the box engine's repeated row reads (warm-up, subtracted rows) touch 4 bytes per
// sample instead of a 32-byte sector.  RPC rows per thread, loads issued before stores.
// grid (ceil(w/256), ceil(h/RPC), planes).
template <int RPC>
__global__ void __launch_bounds__(256) subsample_nearest_kernel(SubParams P) {
    const int x = blockIdx.x * blockDim.x + threadIdx.x;
    if (x >= P.w) return;
    const size_t plane = blockIdx.z;
    const float* src = P.src + plane * (size_t)P.H * P.W + (size_t)x * P.s;
    float* dst = P.dst + plane * (size_t)P.h * P.w + x;
    const int y0 = blockIdx.y * RPC;
    float v[RPC];
#pragma unroll
    for (int k = 0; k < RPC; ++k)
        if (y0 + k < P.h) v[k] = __ldg(src + (size_t)(y0 + k) * P.s * P.W);
#pragma unroll
    for (int k = 0; k < RPC; ++k)
        if (y0 + k < P.h) dst[(size_t)(y0 + k) * P.w] = v[k];
}

// ------------------------------------------------------------------ K1 / K3: strip box filter

template <int MODE, int CI, int CP>
struct StripTraits;

// Statistics of Alg.2 step 2 for gray guidance, per low-res pixel:
//   [0] I', [1] I'I', [2+c] p'_c, [2+CP+c] I'p'_c.
template <int CP>
struct StripTraits<MODE_STATS, 1, CP> {
    static constexpr int NIN = 1 + CP;
    static constexpr int NMAP = 2 + 2 * CP;
    static constexpr int NOUT = 2 * CP;
    __device__ static void products(const float* v, double* pr) {
        const double I = (double)v[0];
        pr[0] = I;
        pr[1] = I * I;  // exact: a float product fits in a double
#pragma unroll
        for (int c = 0; c < CP; ++c) {
            const double p = (double)v[1 + c];
            pr[2 + c] = p;
            pr[2 + CP + c] = I * p;
        }
    }
};

// Color guidance: [0..2] I'_j, [3..8] I'_j I'_k (j<=k: 00 01 02 11 12 22),
//   [9+4c] p'_c, [10+4c+j] I'_j p'_c.
template <int CP>
struct StripTraits<MODE_STATS, 3, CP> {
    static constexpr int NIN = 3 + CP;
    static constexpr int NMAP = 9 + 4 * CP;
    static constexpr int NOUT = 4 * CP;
    __device__ static void products(const float* v, double* pr) {
        const double I0 = v[0], I1 = v[1], I2 = v[2];
        pr[0] = I0; pr[1] = I1; pr[2] = I2;
        pr[3] = I0 * I0; pr[4] = I0 * I1; pr[5] = I0 * I2;
        pr[6] = I1 * I1; pr[7] = I1 * I2; pr[8] = I2 * I2;
#pragma unroll
        for (int c = 0; c < CP; ++c) {
            const double p = (double)v[3 + c];
            pr[9 + 4 * c] = p;
            pr[10 + 4 * c] = I0 * p;
            pr[11 + 4 * c] = I1 * p;
            pr[12 + 4 * c] = I2 * p;
        }
    }
};

// Step 5: the box of the (CI+1)*CP coefficient maps themselves.
template <int CI, int CP>
struct StripTraits<MODE_MEAN, CI, CP> {
    static constexpr int NIN = (CI + 1) * CP;
    static constexpr int NMAP = NIN;
    static constexpr int NOUT = NIN;
    __device__ static void products(const float* v, double* pr) {
#pragma unroll
        for (int m = 0; m < NMAP; ++m) pr[m] = (double)v[m];
    }
};

struct StripParams {
    // Input sample (y, x) of plane j of image b is at src[b*img + j*plane + y*row + x*col];
    // all in-image offsets fit in 32 bits (validated on the host).
    // STATS: srcI = I (or I' planes), srcP = p (or p' planes); MEAN: srcI = coefficient maps.
    const float* srcI;
    const float* srcP;
    long long imgI, imgP;
    int planeI, planeP;
    int row, col;           // row pitch and column stride of a sample
    float* dst;             // [img][(CI+1)CP][h][w]
    int h, w, R;            // low-res dims and radius r'
    int TW, TH;             // output columns per strip, output rows per segment
    int VP;                 // padded fp64 row length in shared memory: NT + 2R + K + 1
    double eps;
    // MEAN only: the written maps are k1 * mean + k0 on the diagonal a maps (a_c for guide
    // channel c), k1 * mean otherwise -- the detail-enhancement fold (fgf_enhance_ws);
    // k1 = 1, k0 = 0 writes the means unchanged.
    float k1, k0;
};

// Rows per batch G (each warp slides along one row of a batch), odd run length K, smem.
// G_ / MINB_ override the defaults (development microbenchmark).
template <int MODE, int CI, int CP, int NT, int G_ = 0, int MINB_ = 0>
struct StripConfig {
    using T = StripTraits<MODE, CI, CP>;
    static constexpr int NMAP = T::NMAP;
    static constexpr int NOUT = T::NOUT;
    static constexpr int NW = NT / 32;
    static constexpr int VPMAX = NT == 256 ? 448 : 992;         // worst-case padded row
    static constexpr int ROWB = NMAP * VPMAX * 8 + NOUT * NT * 4;
    static constexpr int G0 = (160 * 1024) / ROWB;
    static constexpr int G1 = G0 >= 8 ? 8 : (G0 >= 4 ? 4 : (G0 >= 2 ? 2 : 1));
    static constexpr int G2 = (NMAP <= 6 && G1 > 4) ? 4 : G1;    // favour occupancy (measured)
    static constexpr int G = G_ ? G_ : (G2 > NW ? NW : G2);
    static constexpr int WPR = NW / G;                           // warps per row
    static constexpr int K = G == 8 ? 9 : (G == 4 ? 5 : (G == 2 ? 3 : 1));
    static constexpr int WB = T::NIN <= 4 ? 8 : (T::NIN <= 8 ? 4 : 2);
    static constexpr int MINB = MINB_ ? MINB_ : (NMAP <= 6 ? (NT == 256 ? 4 : 2) : 1);
    // dynamic smem for padded row length VP
    static size_t smem(int VP) {
        return (size_t)G * NMAP * VP * 8 + (size_t)G * NOUT * NT * 4 + (size_t)NT * 8;
    }
};

// Epilogue of steps 3-4; writes NOUT values at dst[m * ostride].
template <int MODE, int CI, int CP>
struct StripEpilogue;

// Gray: a = cov/(max(var,0)+eps), b = mean_p - a mean_I (Eq.2-3, R8).
template <int CP>
struct StripEpilogue<MODE_STATS, 1, CP> {
    __device__ static void emit(const double* S, double inv, const StripParams& P, float* dst,
                                int ostride) {
        const double eps = P.eps;
        // The cancellations (var_I, cov_Ip: P:78-79) are formed in fp64; the quotient and b
        // (Eq.2-3) are well conditioned and are formed in fp32.
        const double mI = S[0] * inv;
        double var = fma(-mI, mI, S[1] * inv);       // var_I
        var = var < 0.0 ? 0.0 : var;                 // R8
        const float rden = __frcp_rn((float)(var + eps));
        const float mIf = (float)mI;
#pragma unroll
        for (int c = 0; c < CP; ++c) {
            const double mp = S[2 + c] * inv;
            const double cov = fma(-mI, mp, S[2 + CP + c] * inv);   // cov_Ip
            const float a = (float)cov * rden;                    // Eq.2 / P:80
            dst[(2 * c) * ostride] = a;
            dst[(2 * c + 1) * ostride] = fmaf(-a, mIf, (float)mp);  // Eq.3 / P:81
        }
    }
};

// Color (R9): a_c = (Sigma + eps U)^-1 v_c by the closed-form symmetric adjugate,
// v_c = corr_Ip_c - mu p_bar_c, b_c = p_bar_c - a_c^T mu; all fp64.
template <int CP>
struct StripEpilogue<MODE_STATS, 3, CP> {
    __device__ static void emit(const double* S, double inv, const StripParams& P, float* dst,
                                int ostride) {
        const double eps = P.eps;
        const double m0 = S[0] * inv, m1 = S[1] * inv, m2 = S[2] * inv;
        const double s00 = S[3] * inv - m0 * m0 + eps;
        const double s01 = S[4] * inv - m0 * m1;
        const double s02 = S[5] * inv - m0 * m2;
        const double s11 = S[6] * inv - m1 * m1 + eps;
        const double s12 = S[7] * inv - m1 * m2;
        const double s22 = S[8] * inv - m2 * m2 + eps;
        const double c00 = s11 * s22 - s12 * s12;
        const double c01 = s02 * s12 - s01 * s22;
        const double c02 = s01 * s12 - s02 * s11;
        const double c11 = s00 * s22 - s02 * s02;
        const double c12 = s01 * s02 - s00 * s12;
        const double c22 = s00 * s11 - s01 * s01;
        const double idet = 1.0 / (s00 * c00 + s01 * c01 + s02 * c02);
#pragma unroll
        for (int c = 0; c < CP; ++c) {
            const double mp = S[9 + 4 * c] * inv;
            const double v0 = S[10 + 4 * c] * inv - m0 * mp;
            const double v1 = S[11 + 4 * c] * inv - m1 * mp;
            const double v2 = S[12 + 4 * c] * inv - m2 * mp;
            const double a0 = (c00 * v0 + c01 * v1 + c02 * v2) * idet;
            const double a1 = (c01 * v0 + c11 * v1 + c12 * v2) * idet;
            const double a2 = (c02 * v0 + c12 * v1 + c22 * v2) * idet;
            const double b = mp - (a0 * m0 + a1 * m1 + a2 * m2);
            float* d = dst + (4 * c) * ostride;
            d[0] = (float)a0;
            d[ostride] = (float)a1;
            d[2 * ostride] = (float)a2;
            d[3 * ostride] = (float)b;
        }
    }
};

template <int CI, int CP>
struct StripEpilogue<MODE_MEAN, CI, CP> {
    __device__ static void emit(const double* S, double inv, const StripParams& P, float* dst,
                                int ostride) {
#pragma unroll
        for (int m = 0; m < (CI + 1) * CP; ++m) {
            const int c = m / (CI + 1), j = m - c * (CI + 1);
            dst[m * ostride] = fmaf(P.k1, (float)(S[m] * inv), j == c ? P.k0 : 0.0f);
        }
    }
};

// Loads the NIN inputs of one row for this thread's column (32-bit in-image offsets).
template <int MODE, int CI, int CP>
__device__ __forceinline__ void load_row(const float* bI, const float* bP, int off, int planeI,
                                         int planeP, float* v) {
    using T = StripTraits<MODE, CI, CP>;
    if (MODE == MODE_STATS) {
#pragma unroll
        for (int j = 0; j < CI; ++j) v[j] = __ldg(bI + (off + j * planeI));
#pragma unroll
        for (int c = 0; c < CP; ++c) v[CI + c] = __ldg(bP + (off + c * planeP));
    } else {
#pragma unroll
        for (int m = 0; m < T::NIN; ++m) v[m] = __ldg(bI + (off + m * planeI));
    }
}

// grid (strips, segments, images); block NT.
template <int MODE, int CI, int CP, int NT, int G_ = 0, int MINB_ = 0>
__global__ void __launch_bounds__(NT, (StripConfig<MODE, CI, CP, NT, G_, MINB_>::MINB)) box_strip_kernel(StripParams P) {
    using T = StripTraits<MODE, CI, CP>;
    using C = StripConfig<MODE, CI, CP, NT, G_, MINB_>;
    constexpr int NMAP = T::NMAP;
    constexpr int NIN = T::NIN;
    constexpr int NOUT = T::NOUT;
    constexpr int G = C::G;
    constexpr int K = C::K;
    extern __shared__ double smem_d[];
    const int VP = P.VP;
    double* Vs = smem_d;                                                  // [G][NMAP][VP]
    float* Os = reinterpret_cast<float*>(Vs + (size_t)G * NMAP * VP);      // [G][NOUT][NT]
    double* invx = reinterpret_cast<double*>(Os + (size_t)G * NOUT * NT);  // [NT]

    const int tid = threadIdx.x;
    const int img = blockIdx.z;
    const int h = P.h, w = P.w, R = P.R;
    const int n = h * w;
    const int x0 = blockIdx.x * P.TW;
    const int xe = min(w, x0 + P.TW);
    const int y0 = blockIdx.y * P.TH;
    const int ye = min(h, y0 + P.TH);
    const int xs0 = max(0, x0 - R);
    const int ncol = min(w, xe + R) - xs0;
    const int ocn = xe - x0;                 // output columns of this strip
    const int cbase = x0 - xs0;              // local column of output column 0
    const bool colthr = tid < ncol;
    const int offc = (xs0 + (colthr ? tid : 0)) * P.col;
    const int row = P.row, planeI = P.planeI, planeP = P.planeP;
    const float* bI = P.srcI + img * P.imgI;
    const float* bP = (MODE == MODE_STATS) ? P.srcP + img * P.imgP : bI;
    float* dst = P.dst + (size_t)img * NOUT * n + x0;

    // Zero the padded column-sum rows once: the pads make every horizontal window read
    // in-bounds, and zeros contribute nothing, so sums equal the clipped sums (R1).
    for (int i = tid; i < G * NMAP * VP; i += NT) Vs[i] = 0.0;
    // 1 / (horizontal in-bounds count) per output column.
    if (tid < ocn) {
        const int c = cbase + tid;
        invx[tid] = 1.0 / (double)(min(ncol - 1, c + R) - max(0, c - R) + 1);
    }

    // Running vertical window sums of this thread's column (fp64; products of two floats are
    // exact in fp64).
    double acc[NMAP];
#pragma unroll
    for (int m = 0; m < NMAP; ++m) acc[m] = 0.0;

    // Warm-up: the window of "row y0-1", rows [y0-R-1, y0+R-1] clipped; WB rows per round.
    if (colthr) {
        constexpr int WB = C::WB;
        const int wa = max(0, y0 - R - 1), wb = min(h - 1, y0 + R - 1);
        for (int y = wa; y <= wb; y += WB) {
            float v[WB][NIN];
#pragma unroll
            for (int k = 0; k < WB; ++k)
                if (y + k <= wb) load_row<MODE, CI, CP>(bI, bP, (y + k) * row + offc, planeI, planeP, v[k]);
#pragma unroll
            for (int k = 0; k < WB; ++k) {
                if (y + k <= wb) {
                    double pr[NMAP];
                    T::products(v[k], pr);
#pragma unroll
                    for (int m = 0; m < NMAP; ++m) acc[m] += pr[m];
                }
            }
        }
    }

    // Horizontal-phase mapping: warp -> row hg of the batch; the WPR warps of a row split it
    // into 32*WPR runs of K (odd) consecutive output columns, so the 16 lanes of a half-warp
    // read 16 distinct fp64 banks.
    const int warp = tid >> 5, lane = tid & 31;
    const int hg = warp % G;
    const int oc0 = ((warp / G) * 32 + lane) * K;

    // Software pipeline: va/vs hold the add/subtract rows of the current batch.  Branch-free:
    // row indices are clamped into the image and rows that must not contribute (beyond the
    // bottom, before the top, past the segment) are zeroed, which adds exactly nothing.
    float va[G][NIN], vs[G][NIN];
    auto load_batch = [&](int yb) {
#pragma unroll
        for (int g = 0; g < G; ++g) {
            const int yo = yb + g;
            const bool oka = yo < ye && yo + R < h;
            const bool oks = yo < ye && yo - R - 1 >= 0;
            load_row<MODE, CI, CP>(bI, bP, min(yo + R, h - 1) * row + offc, planeI, planeP, va[g]);
            load_row<MODE, CI, CP>(bI, bP, max(yo - R - 1, 0) * row + offc, planeI, planeP, vs[g]);
#pragma unroll
            for (int k = 0; k < NIN; ++k) {
                va[g][k] = oka ? va[g][k] : 0.0f;
                vs[g][k] = oks ? vs[g][k] : 0.0f;
            }
        }
    };
    if (colthr) load_batch(y0);

    int prev_rows = 0;       // rows staged in Os by the previous batch, not yet stored
    int prev_yb = 0;
    for (int yb = y0; yb < ye; yb += G) {
        // ---- column phase: slide the vertical windows of the batch's rows, snapshot.
        if (colthr) {
#pragma unroll
            for (int g = 0; g < G; ++g) {
                double pa[NMAP], ps[NMAP];
                T::products(va[g], pa);
                T::products(vs[g], ps);
                double* vrow = Vs + (size_t)g * NMAP * VP + R + tid;
#pragma unroll
                for (int m = 0; m < NMAP; ++m) {
                    acc[m] += pa[m] - ps[m];
                    vrow[m * VP] = acc[m];
                }
            }
        }
        // ---- coalesced store of the previous batch's staged outputs (one column per thread).
        if (tid < ocn) {
            for (int g = 0; g < prev_rows; ++g) {
                float* drow = dst + (size_t)(prev_yb + g) * w + tid;
                const float* orow = Os + (size_t)g * NOUT * NT + tid;
#pragma unroll
                for (int m = 0; m < NOUT; ++m) drow[(size_t)m * n] = orow[m * NT];
            }
        }
        __syncthreads();

        // ---- prefetch the next batch (in flight during the horizontal phase).
        if (colthr && yb + G < ye) load_batch(yb + G);

        // ---- horizontal phase: branch-free sliding window along each snapshotted row.
        const int yo = yb + hg;
        if (yo < ye && oc0 < ocn) {
            const double* vr = Vs + (size_t)hg * NMAP * VP + R + cbase + oc0;  // local col of oc0
            const double invy = 1.0 / (double)(min(h - 1, yo + R) - max(0, yo - R) + 1);
            double S[NMAP];
#pragma unroll
            for (int m = 0; m < NMAP; ++m) S[m] = 0.0;
#pragma unroll 4
            for (int k = -R; k <= R; ++k) {
#pragma unroll
                for (int m = 0; m < NMAP; ++m) S[m] += vr[m * VP + k];
            }
            float* orow = Os + (size_t)hg * NOUT * NT + oc0;
#pragma unroll
            for (int i = 0; i < K; ++i) {
                if (oc0 + i < ocn)
                    StripEpilogue<MODE, CI, CP>::emit(S, invx[oc0 + i] * invy, P, orow + i, NT);
                if (i + 1 < K) {
#pragma unroll
                    for (int m = 0; m < NMAP; ++m) S[m] += vr[m * VP + i + R + 1] - vr[m * VP + i - R];
                }
            }
        }
        prev_rows = min(G, ye - yb);
        prev_yb = yb;
        __syncthreads();
    }
    if (tid < ocn) {
        for (int g = 0; g < prev_rows; ++g) {
            float* drow = dst + (size_t)(prev_yb + g) * w + tid;
            const float* orow = Os + (size_t)g * NOUT * NT + tid;
#pragma unroll
            for (int m = 0; m < NOUT; ++m) drow[(size_t)m * n] = orow[m * NT];
        }
    }
}

// ------------------------------------------------------------------ K4: upsample + output

struct OutParams {
    const float* I;        // [img][CI][H][W]   (H rows of the image, or of a row band)
    const float* M;        // [img][(CI+1)CP][hm][w] mean maps (hm low-res rows)
    float* q;              // [img][CP][H][W]
    int H, W, hm, w;       // local buffer geometry
    int Hg, hg;            // global full-res / low-res heights (the vertical map, R5)
    int Yoff, yoff;        // global row of local row 0 of I/q, and of the maps buffer
    int TR;                // full-resolution rows walked by each thread
};

// R5: source coordinate of destination index d, resize n_src -> n_dst, exactly in
// integers: c = ((2d+1) n_src - n_dst) / (2 n_dst), clamped to [0, n_src-1].
__device__ __forceinline__ void src_coord(int d, int n_src, int n_dst, int& i0, int& i1,
                                          float& f) {
    if ((long long)(2 * n_dst + 1) * n_src < (1LL << 31)) {   // exact in 32-bit arithmetic
        const int num = (2 * d + 1) * n_src - n_dst;
        const int den = 2 * n_dst;
        if (num <= 0) {
            i0 = 0;
            f = 0.0f;
        } else {
            const int q = (int)((unsigned)num / (unsigned)den);
            if (q >= n_src - 1) {
                i0 = n_src - 1;
                f = 0.0f;
            } else {
                i0 = q;
                f = (float)(num - q * den) / (float)den;
            }
        }
        i1 = min(i0 + 1, n_src - 1);
        return;
    }
    const long long num = (long long)(2 * d + 1) * n_src - n_dst;
    const long long den = 2LL * n_dst;
    if (num <= 0) {
        i0 = 0;
        f = 0.0f;
    } else {
        const long long q = num / den;
        if (q >= n_src - 1) {
            i0 = n_src - 1;
            f = 0.0f;
        } else {
            i0 = (int)q;
            f = (float)(num - q * den) / (float)den;
        }
    }
    i1 = min(i0 + 1, n_src - 1);
}

template <int PX>
struct VecT;
template <>
struct VecT<1> {
    using T = float;
    __device__ static T ld(const float* p) { return __ldcs(p); }
    __device__ static void st(float* p, const float* v) { __stcs(p, v[0]); }
    __device__ static float get(const T& v, int) { return v; }
};
template <>
struct VecT<2> {
    using T = float2;
    __device__ static T ld(const float* p) { return __ldcs(reinterpret_cast<const float2*>(p)); }
    __device__ static void st(float* p, const float* v) {
        __stcs(reinterpret_cast<float2*>(p), make_float2(v[0], v[1]));
    }
    __device__ static float get(const T& v, int i) { return i == 0 ? v.x : v.y; }
};
template <>
struct VecT<4> {
    using T = float4;
    __device__ static T ld(const float* p) { return __ldcs(reinterpret_cast<const float4*>(p)); }
    __device__ static void st(float* p, const float* v) {
        __stcs(reinterpret_cast<float4*>(p), make_float4(v[0], v[1], v[2], v[3]));
    }
    __device__ static float get(const T& v, int i) {
        return i == 0 ? v.x : (i == 1 ? v.y : (i == 2 ? v.z : v.w));
    }
};

// Column walker.  Each thread owns PX consecutive pixels of a row and walks the TR rows of
// its CTA's band.  Their horizontal source coordinates are fixed, so the horizontally
// interpolated coefficient rows H0 = Hx(y0), H1 = Hx(y1) live in registers and are
// refreshed only when the low-res row pair changes (every ~s rows; the row table is in
// shared memory and the test is a warp vote, so the branch is CTA-uniform).  The low-res
// coefficient rows the band touches are staged into shared memory once per CTA (coalesced
// loads issued right after the first image rows), so refreshes never wait on L2.  Per pixel
// and map the upsample is then A = H0 + fy (H1 - H0) and q_c = sum_j A_{c,j} I_j + A_{c,CI}
// (P:84-86).  Full-resolution rows of I are prefetched U rows ahead in a rolling register
// ring with streaming (evict-first) loads; q is written with streaming stores.
// S1 (s = 1, h = H, w = W): the upsample is the identity, A = M; the maps are streamed with I.
// grid (ceil(W / (256 PX)), ceil(H / TR), images), block 256, TR <= kMaxTR,
// dynamic smem nrl * NC * ncl floats (host-computed maxima; none when S1).
constexpr int kMaxTR = 128;

// Defaults measured with tools/k4_bench.cu (profiles/round1/k4_microbench.txt): more
// resident warps beat deeper per-thread prefetch; 4 CTAs/SM is the register limit before
// spills.
template <int CI, int CP, int PX>
struct OutCfg {
    static constexpr int NC = (CI + 1) * CP;
    static constexpr int U0 = 8 / (CI * PX);
    static constexpr int U = U0 > 8 ? 8 : (U0 < 2 ? 2 : U0);
    static constexpr int MINB = NC * PX <= 8 ? 4 : 2;
};

// U_ / MINB_ override the defaults (rows in flight per thread, CTAs per SM for registers).
// ABL: ablation switch for the development microbenchmark (0 = the real kernel; 1 = skip
// the coefficient refresh; 2 = q = I copy in the same access pattern).
template <int CI, int CP, int PX, bool S1, int U_ = 0, int MINB_ = 0, int ABL = 0>
__global__ void __launch_bounds__(256, (MINB_ ? MINB_ : OutCfg<CI, CP, PX>::MINB)) output_kernel(OutParams P) {
    constexpr int NC = OutCfg<CI, CP, PX>::NC;
    constexpr int U = U_ ? U_ : OutCfg<CI, CP, PX>::U;
    constexpr int NL = S1 ? CI + NC : CI;        // planes streamed per row
    using V = VecT<PX>;
    using VT = typename V::T;
    __shared__ int s_ya[kMaxTR];
    __shared__ int s_y1[kMaxTR];
    __shared__ float s_fy[kMaxTR];
    extern __shared__ float Ms[];                // [nrl][NC][ncl]
    const int H = P.H, W = P.W, h = P.hm, w = P.w;
    const int Y0 = blockIdx.y * P.TR;
    const int nrows = min(P.TR, H - Y0);
    const int X0 = blockIdx.x * 256 * PX;
    const bool act = X0 + threadIdx.x * PX < W;
    const int X = act ? X0 + threadIdx.x * PX : X0;
    const int img = blockIdx.z;
    const size_t N = (size_t)H * W, n = (size_t)h * w;
    const float* Ip = P.I + (size_t)img * CI * N + (size_t)Y0 * W + X;
    float* qp = P.q + (size_t)img * CP * N + (size_t)Y0 * W + X;
    const float* Mb = P.M + (size_t)img * NC * n;
    // S1 only: the maps have the image's geometry, shifted by the band offsets
    const float* Mp = Mb + (size_t)(P.Yoff + Y0 - P.yoff) * W + X;

    // Plane j of the streamed row: I planes, then (S1) the coefficient maps.
    auto plane_ptr = [&](const float* base_row, int j) -> const float* {
        return (!S1 || j < CI) ? base_row + (size_t)j * N : Mp + (base_row - Ip) + (size_t)(j - CI) * n;
    };

    // Issue the first U rows before anything else.
    VT cur[U][NL];
#pragma unroll
    for (int u = 0; u < U; ++u)
        if (act && u < nrows)
#pragma unroll
            for (int j = 0; j < NL; ++j) cur[u][j] = V::ld(plane_ptr(Ip + (size_t)u * W, j));

    int oa[PX], ob[PX];
    float fx[PX];
    int ylo = 0, ncl = 0;
    if (!S1) {
        // Row table and the low-res rectangle [ylo, yhi] x [xlo, xhi] this CTA touches.
        // (global vertical map, then local to the maps buffer)
        for (int t = threadIdx.x; t < nrows; t += 256) {
            int ya, yb;
            float fy;
            src_coord(P.Yoff + Y0 + t, P.hg, P.Hg, ya, yb, fy);
            s_ya[t] = ya - P.yoff;
            s_y1[t] = yb - P.yoff;
            s_fy[t] = fy;
        }
        int yd, yhi, xlo, xd, xhi;
        float fd;
        src_coord(P.Yoff + Y0, P.hg, P.Hg, ylo, yd, fd);
        src_coord(P.Yoff + Y0 + nrows - 1, P.hg, P.Hg, yd, yhi, fd);
        ylo -= P.yoff;
        yhi -= P.yoff;
        src_coord(X0, w, W, xlo, xd, fd);
        src_coord(min(W, X0 + 256 * PX) - 1, w, W, xd, xhi, fd);
        const int nrl = yhi - ylo + 1;
        ncl = xhi - xlo + 1;
        // one warp per (row, map) line of the rectangle, lanes along the columns
        for (int rm = threadIdx.x >> 5; rm < nrl * NC; rm += 8) {
            const int rr = rm / NC, m = rm - rr * NC;
            const float* src = Mb + (size_t)m * n + (size_t)(ylo + rr) * w + xlo;
            float* d = Ms + (size_t)rm * ncl;
            for (int xx = threadIdx.x & 31; xx < ncl; xx += 32) d[xx] = __ldg(src + xx);
        }
#pragma unroll
        for (int i = 0; i < PX; ++i) {
            src_coord(min(X + i, W - 1), w, W, oa[i], ob[i], fx[i]);
            oa[i] -= xlo;      // local columns in the staged rectangle
            ob[i] -= xlo;
        }
        __syncthreads();
    }

    const float* Ipf = Ip + (size_t)U * W;
    int cy = -2, cy1 = -2;
    float H0[NC][PX], H1[NC][PX], D[NC][PX];
    auto hrow = [&](int y, float (&out)[NC][PX]) {
        const float* mr = Ms + (size_t)(y - ylo) * NC * ncl;
#pragma unroll
        for (int m = 0; m < NC; ++m)
#pragma unroll
            for (int i = 0; i < PX; ++i) {
                const float va = mr[m * ncl + oa[i]], vb = mr[m * ncl + ob[i]];
                out[m][i] = fmaf(fx[i], vb - va, va);
            }
    };
    for (int rb0 = 0; rb0 < nrows; rb0 += U) {
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int t = rb0 + u;
            if (t < nrows) {
                float fy = 0.0f;
                if (!S1) {
                    const int ya = s_ya[t];
                    fy = s_fy[t];
                    if (ABL == 0 && __any_sync(0xffffffffu, ya != cy)) {   // CTA-uniform branch
                        if (act) {
                            if (ya == cy1) {
#pragma unroll
                                for (int m = 0; m < NC; ++m)
#pragma unroll
                                    for (int i = 0; i < PX; ++i) H0[m][i] = H1[m][i];
                            } else {
                                hrow(ya, H0);
                            }
                            cy1 = s_y1[t];
                            hrow(cy1, H1);
#pragma unroll
                            for (int m = 0; m < NC; ++m)
#pragma unroll
                                for (int i = 0; i < PX; ++i) D[m][i] = H1[m][i] - H0[m][i];
                        }
                        cy = ya;
                    }
                }
                if (!act) continue;
                if (ABL != 0 && t == 0) {
#pragma unroll
                    for (int m = 0; m < NC; ++m)
#pragma unroll
                        for (int i = 0; i < PX; ++i) { H0[m][i] = 0.5f; D[m][i] = 0.25f; }
                }
#pragma unroll
                for (int c = 0; c < CP; ++c) {
                    const int mb = c * (CI + 1);
                    float o[PX];
#pragma unroll
                    for (int i = 0; i < PX; ++i) {
                        if (ABL == 2) { o[i] = V::get(cur[u][0], i); continue; }
                        float acc;
                        if (S1) {
                            acc = V::get(cur[u][CI + mb + CI], i);
#pragma unroll
                            for (int j = 0; j < CI; ++j)
                                acc = fmaf(V::get(cur[u][CI + mb + j], i), V::get(cur[u][j], i), acc);
                        } else {
                            acc = fmaf(fy, D[mb + CI][i], H0[mb + CI][i]);
#pragma unroll
                            for (int j = 0; j < CI; ++j)
                                acc = fmaf(fmaf(fy, D[mb + j][i], H0[mb + j][i]), V::get(cur[u][j], i), acc);
                        }
                        o[i] = acc;
                    }
                    V::st(qp + c * N, o);
                }
                qp += W;
                // Rolling prefetch: this register slot now takes row t + U.
                if (t + U < nrows)
#pragma unroll
                    for (int j = 0; j < NL; ++j) cur[u][j] = V::ld(plane_ptr(Ipf, j));
                Ipf += W;
            }
        }
    }
}

// ------------------------------------------------------------------ K4, cp.async ring
//
// The column walker with its U-row prefetch of I kept in SHARED memory instead of registers:
// each thread copies its own PX pixels of row t+U with cp.async (LDGSTS, L2 -> smem, no
// register held while in flight) into a per-thread ring slot, one commit group per row, and
// waits with cp.async.wait_group(U-1) before consuming row t.  With ~60 registers the SM
// keeps 4 CTAs resident and U = 8 rows x 16 B x 1024 threads = 128 KB of I in flight.

__device__ __forceinline__ void cp_async4(float* dst, const float* src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"((uint32_t)__cvta_generic_to_shared(dst)),
                 "l"(src)
                 : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }

template <int BYTES>
__device__ __forceinline__ void cp_async_px(void* dst, const float* src) {
    const uint32_t d = (uint32_t)__cvta_generic_to_shared(dst);
    if (BYTES == 16)
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(d), "l"(src) : "memory");
    else if (BYTES == 8)
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(d), "l"(src) : "memory");
    else
        asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(d), "l"(src) : "memory");
}
template <int N>
__device__ __forceinline__ void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

template <int CI, int CP, int PX>
struct AsyncCfg {
    static constexpr int NC = (CI + 1) * CP;
    static constexpr int U = 8;                                  // rows in flight (power of 2)
    static constexpr int MINB = NC * PX <= 8 ? 4 : 2;
    static constexpr size_t RING_BYTES = (size_t)U * CI * 256 * PX * 4;
};

template <int CI, int CP, int PX>
__global__ void __launch_bounds__(256, (AsyncCfg<CI, CP, PX>::MINB)) output_async_kernel(OutParams P) {
    using C = AsyncCfg<CI, CP, PX>;
    constexpr int NC = C::NC;
    constexpr int U = C::U;
    using V = VecT<PX>;
    using VT = typename V::T;
    __shared__ int s_ya[kMaxTR];
    __shared__ int s_y1[kMaxTR];
    __shared__ float s_fy[kMaxTR];
    extern __shared__ __align__(16) float smx[];
    VT* ring = reinterpret_cast<VT*>(smx);                        // [U][CI][256]
    float* Ms = smx + C::RING_BYTES / 4;                          // [nrl][NC][ncl]
    const int H = P.H, W = P.W, h = P.hm, w = P.w;
    const int tid = threadIdx.x;
    const int Y0 = blockIdx.y * P.TR;
    const int nrows = min(P.TR, H - Y0);
    const int X0 = blockIdx.x * 256 * PX;
    const bool act = X0 + tid * PX < W;
    const int X = act ? X0 + tid * PX : X0;
    const int img = blockIdx.z;
    const size_t N = (size_t)H * W, n = (size_t)h * w;
    const float* Ip = P.I + (size_t)img * CI * N + (size_t)Y0 * W + X;
    float* qp = P.q + (size_t)img * CP * N + (size_t)Y0 * W + X;
    const float* Mb = P.M + (size_t)img * NC * n;

    // Issue the first U rows (one commit group per row, empty groups keep the count uniform).
#pragma unroll
    for (int u = 0; u < U; ++u) {
        if (act && u < nrows)
#pragma unroll
            for (int j = 0; j < CI; ++j)
                cp_async_px<PX * 4>(&ring[(u * CI + j) * 256 + tid], Ip + j * N + (size_t)u * W);
        cp_async_commit();
    }

    // Row table and staged low-res rectangle (as in output_kernel).
    for (int t = tid; t < nrows; t += 256) {
        int ya, yb;
        float fy;
        src_coord(P.Yoff + Y0 + t, P.hg, P.Hg, ya, yb, fy);
        s_ya[t] = ya - P.yoff;
        s_y1[t] = yb - P.yoff;
        s_fy[t] = fy;
    }
    int ylo, yd, yhi, xlo, xd, xhi;
    float fd;
    src_coord(P.Yoff + Y0, P.hg, P.Hg, ylo, yd, fd);
    src_coord(P.Yoff + Y0 + nrows - 1, P.hg, P.Hg, yd, yhi, fd);
    ylo -= P.yoff;
    yhi -= P.yoff;
    src_coord(X0, w, W, xlo, xd, fd);
    src_coord(min(W, X0 + 256 * PX) - 1, w, W, xd, xhi, fd);
    const int nrl = yhi - ylo + 1, ncl = xhi - xlo + 1;
    for (int rm = tid >> 5; rm < nrl * NC; rm += 8) {
        const int rr = rm / NC, m = rm - rr * NC;
        const float* src = Mb + (size_t)m * n + (size_t)(ylo + rr) * w + xlo;
        float* d = Ms + (size_t)rm * ncl;
        for (int xx = tid & 31; xx < ncl; xx += 32) d[xx] = __ldg(src + xx);
    }
    int oa[PX], ob[PX];
    float fx[PX];
#pragma unroll
    for (int i = 0; i < PX; ++i) {
        src_coord(min(X + i, W - 1), w, W, oa[i], ob[i], fx[i]);
        oa[i] -= xlo;
        ob[i] -= xlo;
    }
    __syncthreads();

    int cy = -2, cy1 = -2;
    float H0[NC][PX], H1[NC][PX], D[NC][PX];
    auto hrow = [&](int y, float (&out)[NC][PX]) {
        const float* mr = Ms + (size_t)(y - ylo) * NC * ncl;
#pragma unroll
        for (int m = 0; m < NC; ++m)
#pragma unroll
            for (int i = 0; i < PX; ++i) {
                const float va = mr[m * ncl + oa[i]], vb = mr[m * ncl + ob[i]];
                out[m][i] = fmaf(fx[i], vb - va, va);
            }
    };
    const float* Ipf = Ip + (size_t)U * W;
    for (int t = 0; t < nrows; ++t) {
        const int ya = s_ya[t];
        const float fy = s_fy[t];
        if (__any_sync(0xffffffffu, ya != cy)) {   // CTA-uniform branch
            if (act) {
                if (ya == cy1) {
#pragma unroll
                    for (int m = 0; m < NC; ++m)
#pragma unroll
                        for (int i = 0; i < PX; ++i) H0[m][i] = H1[m][i];
                } else {
                    hrow(ya, H0);
                }
                cy1 = s_y1[t];
                hrow(cy1, H1);
#pragma unroll
                for (int m = 0; m < NC; ++m)
#pragma unroll
                    for (int i = 0; i < PX; ++i) D[m][i] = H1[m][i] - H0[m][i];
            }
            cy = ya;
        }
        cp_async_wait<U - 1>();                     // row t has landed in this thread's slot
        const int slot = t & (U - 1);
        if (act) {
            VT iv[CI];
#pragma unroll
            for (int j = 0; j < CI; ++j) iv[j] = ring[(slot * CI + j) * 256 + tid];
#pragma unroll
            for (int c = 0; c < CP; ++c) {
                const int mb = c * (CI + 1);
                float o[PX];
#pragma unroll
                for (int i = 0; i < PX; ++i) {
                    float acc = fmaf(fy, D[mb + CI][i], H0[mb + CI][i]);
#pragma unroll
                    for (int j = 0; j < CI; ++j)
                        acc = fmaf(fmaf(fy, D[mb + j][i], H0[mb + j][i]), V::get(iv[j], i), acc);
                    o[i] = acc;
                }
                V::st(qp + c * N, o);
            }
            // the slot's values are consumed (the stores above depend on them): refill it
            if (t + U < nrows)
#pragma unroll
                for (int j = 0; j < CI; ++j)
                    cp_async_px<PX * 4>(&ring[(slot * CI + j) * 256 + tid], Ipf + j * N);
        }
        cp_async_commit();
        qp += W;
        Ipf += W;
    }
    cp_async_wait<0>();
}

// ------------------------------------------------------------------ K4, persistent
//
// Persistent column walker (s > 1).  The grid is ncb x cpb CTAs (about two per SM); CTA
// (cb, k) owns the 256 PX-pixel column block cb and walks the bands k, k + cpb, ... of all
// images as one continuous stream of rows.  The low-res rectangle and row table of the NEXT
// band are staged with cp.async into the other half of a double buffer while the current
// band streams, and the rolling U-row register prefetch of I runs across band boundaries, so
// neither the staging latency nor a band change ever idles the HBM pipe.


struct PersistParams {
    OutParams o;           // geometry (TR = rows per band)
    int images, ncb, cpb;
    int nrl, ncl;          // staged rectangle capacity (rows, cols)
};

template <int CI, int CP, int PX>
struct PersistCfg {
    static constexpr int NC = (CI + 1) * CP;
    static constexpr int U0 = 32 / (CI * PX);
    static constexpr int U = U0 > 8 ? 8 : (U0 < 2 ? 2 : U0);
    static constexpr int MINB = NC * PX <= 8 ? 2 : 1;
};

template <int CI, int CP, int PX>
__global__ void __launch_bounds__(256, (PersistCfg<CI, CP, PX>::MINB)) output_persist_kernel(PersistParams PP) {
    constexpr int NC = PersistCfg<CI, CP, PX>::NC;
    constexpr int U = PersistCfg<CI, CP, PX>::U;
    using V = VecT<PX>;
    using VT = typename V::T;
    const OutParams& P = PP.o;
    __shared__ int s_ya[2][kMaxTR];
    __shared__ int s_y1[2][kMaxTR];
    __shared__ float s_fy[2][kMaxTR];
    extern __shared__ float Msh[];                    // [2][nrl][NC][ncl]
    const int H = P.H, W = P.W, w = P.w, TR = P.TR;
    const size_t N = (size_t)H * W, n = (size_t)P.hm * w;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int cb = blockIdx.x % PP.ncb;
    const int k0 = blockIdx.x / PP.ncb;
    const int bands = (H + TR - 1) / TR;
    const int items = PP.images * bands;
    if (k0 >= items) return;                           // CTA-uniform
    const int X0 = cb * 256 * PX;
    const bool act = X0 + tid * PX < W;
    const int X = act ? X0 + tid * PX : X0;
    const size_t bufsz = (size_t)PP.nrl * NC * PP.ncl;

    // Horizontal geometry of this column block (fixed for the CTA's lifetime).
    int xlo, xd, xhi;
    float fd;
    src_coord(X0, w, W, xlo, xd, fd);
    src_coord(min(W, X0 + 256 * PX) - 1, w, W, xd, xhi, fd);
    const int ncl = xhi - xlo + 1;
    int oa[PX], ob[PX];
    float fx[PX];
#pragma unroll
    for (int i = 0; i < PX; ++i) {
        src_coord(min(X + i, W - 1), w, W, oa[i], ob[i], fx[i]);
        oa[i] -= xlo;
        ob[i] -= xlo;
    }

    auto band_rows = [&](int item) { return min(TR, H - (item % bands) * TR); };
    // Stage band `item` (row table + low-res rectangle) into buffer `b` (cp.async, no wait).
    int ylo_b[2] = {0, 0};
    auto stage = [&](int item, int b) {
        if (item >= items) return;
        const int img = item / bands, Yb = (item % bands) * TR, nr = band_rows(item);
        for (int t = tid; t < nr; t += 256) {
            int ya, yb;
            float fy;
            src_coord(P.Yoff + Yb + t, P.hg, P.Hg, ya, yb, fy);
            s_ya[b][t] = ya - P.yoff;
            s_y1[b][t] = yb - P.yoff;
            s_fy[b][t] = fy;
        }
        int ylo, yhi, yd2;
        float f2;
        src_coord(P.Yoff + Yb, P.hg, P.Hg, ylo, yd2, f2);
        src_coord(P.Yoff + Yb + nr - 1, P.hg, P.Hg, yd2, yhi, f2);
        ylo -= P.yoff;
        yhi -= P.yoff;
        ylo_b[b] = ylo;
        const float* Mb = P.M + (size_t)img * NC * n + xlo;
        float* dst = Msh + b * bufsz;
        const int nrm = (yhi - ylo + 1) * NC;
        for (int rm = warp; rm < nrm; rm += 8) {
            const int rr = rm / NC, m = rm - rr * NC;
            const float* src = Mb + (size_t)m * n + (size_t)(ylo + rr) * w;
            float* d = dst + (size_t)rm * ncl;
            for (int xx = lane; xx < ncl; xx += 32) cp_async4(d + xx, src + xx);
        }
        cp_async_commit();
    };

    // Band bases: (item) -> pointer to row 0 of the band at this thread's pixels.
    auto I_base = [&](int item) {
        const int img = item / bands, Yb = (item % bands) * TR;
        return P.I + (size_t)img * CI * N + (size_t)Yb * W + X;
    };
    auto q_base = [&](int item) {
        const int img = item / bands, Yb = (item % bands) * TR;
        return P.q + (size_t)img * CP * N + (size_t)Yb * W + X;
    };

    stage(k0, 0);
    cp_async_wait_all();
    __syncthreads();
    stage(k0 + PP.cpb, 1);

    // prefetch cursor (U rows ahead): band item, row pointer, rows left in the band
    int p_item = k0, p_left = band_rows(k0);
    const float* p_ptr = I_base(k0);
    auto p_advance = [&]() {
        p_ptr += W;
        if (--p_left == 0) {
            p_item += PP.cpb;
            if (p_item < items) {
                p_left = band_rows(p_item);
                p_ptr = I_base(p_item);
            }
        }
    };
    VT cur[U][CI];
#pragma unroll
    for (int u = 0; u < U; ++u) {
        if (p_item < items) {
            if (act)
#pragma unroll
                for (int j = 0; j < CI; ++j) cur[u][j] = V::ld(p_ptr + j * N);
            p_advance();
        }
    }

    int c_item = k0, c_t = 0, c_rows = band_rows(k0), buf = 0, cy = -2, cy1 = -2;
    float* c_q = q_base(k0);
    float H0[NC][PX], H1[NC][PX], D[NC][PX];
    auto hrow = [&](int y, float (&out)[NC][PX]) {
        const float* mr = Msh + buf * bufsz + (size_t)(y - ylo_b[buf]) * NC * ncl;
#pragma unroll
        for (int m = 0; m < NC; ++m)
#pragma unroll
            for (int i = 0; i < PX; ++i) {
                const float va = mr[m * ncl + oa[i]], vb = mr[m * ncl + ob[i]];
                out[m][i] = fmaf(fx[i], vb - va, va);
            }
    };
    while (c_item < items) {
#pragma unroll
        for (int u = 0; u < U; ++u) {
            if (c_item < items) {
                if (c_t == 0 && c_item != k0) {
                    // new band: its staging (issued one band ago) must be complete, and every
                    // thread must be done with the old buffer before it is refilled
                    cp_async_wait_all();
                    __syncthreads();
                    buf ^= 1;
                    cy = -2;
                    stage(c_item + PP.cpb, buf ^ 1);
                }
                const int ya = s_ya[buf][c_t];
                const float fy = s_fy[buf][c_t];
                if (__any_sync(0xffffffffu, ya != cy)) {   // CTA-uniform branch
                    if (act) {
                        if (ya == cy1) {
#pragma unroll
                            for (int m = 0; m < NC; ++m)
#pragma unroll
                                for (int i = 0; i < PX; ++i) H0[m][i] = H1[m][i];
                        } else {
                            hrow(ya, H0);
                        }
                        cy1 = s_y1[buf][c_t];
                        hrow(cy1, H1);
#pragma unroll
                        for (int m = 0; m < NC; ++m)
#pragma unroll
                            for (int i = 0; i < PX; ++i) D[m][i] = H1[m][i] - H0[m][i];
                    }
                    cy = ya;
                }
                if (act) {
                    float* qrow = c_q;
#pragma unroll
                    for (int c = 0; c < CP; ++c) {
                        const int mb = c * (CI + 1);
                        float o[PX];
#pragma unroll
                        for (int i = 0; i < PX; ++i) {
                            float acc = fmaf(fy, D[mb + CI][i], H0[mb + CI][i]);
#pragma unroll
                            for (int j = 0; j < CI; ++j)
                                acc = fmaf(fmaf(fy, D[mb + j][i], H0[mb + j][i]), V::get(cur[u][j], i), acc);
                            o[i] = acc;
                        }
                        V::st(qrow + c * N, o);
                    }
                }
                // rolling prefetch: this slot takes the stream row U ahead
                if (p_item < items) {
                    if (act)
#pragma unroll
                        for (int j = 0; j < CI; ++j) cur[u][j] = V::ld(p_ptr + j * N);
                    p_advance();
                }
                c_q += W;
                if (++c_t >= c_rows) {
                    c_t = 0;
                    c_item += PP.cpb;
                    if (c_item < items) {
                        c_rows = band_rows(c_item);
                        c_q = q_base(c_item);
                    }
                }
            }
        }
    }
    cp_async_wait_all();
}

// ------------------------------------------------------------------ K4 (TMA pipeline)
//
// Persistent variant of K4 for 16-byte aligned rows (W % 4 == 0).  The image is cut into
// column blocks of 1024 pixels; every CTA owns one column block (so each thread's four
// horizontal source coordinates are computed once) and walks bands of TR rows of successive
// images.  Thread 0 streams the rows of I into a ring of NSTAGE shared-memory stages with
// 1-D bulk copies (cp.async.bulk, evict-first L2 policy) completing on per-stage mbarriers,
// keeping NSTAGE * RPS rows (>= 96 KB) in flight per SM; the 256 threads read their float4
// from shared memory, apply the register-resident coefficient rows, and stream q out.

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, int count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ uint64_t evict_first_policy() {
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar,
                                         uint64_t pol) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
        " [%0], [%1], %2, [%3], %4;" ::"r"(smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
        : "memory");
}

struct TmaOutParams {
    const float* I;        // [img][CI][H][W]
    const float* M;        // [img][(CI+1)CP][h][w]
    float* q;              // [img][CP][H][W]
    int H, W, h, w;
    int images;            // images in this launch
    int TR;                // rows per band
    int ncb;               // column blocks of 1024 px
    int cpb;               // CTAs per column block (gridDim.x = ncb * cpb)
};

template <int CI, int CP>
struct TmaCfg {
    static constexpr int NC = (CI + 1) * CP;
    static constexpr int RPS = CI == 1 ? 4 : 2;        // rows per stage
    static constexpr int NSTAGE = CI == 1 ? 8 : 6;
    static constexpr int ROWF = 1024;                   // floats per row segment
    static constexpr size_t STAGE_FLOATS = (size_t)RPS * CI * ROWF;
    static constexpr size_t SMEM = NSTAGE * STAGE_FLOATS * 4 + NSTAGE * 8;
};

template <int CI, int CP>
__global__ void __launch_bounds__(256, 1) output_tma_kernel(TmaOutParams P) {
    using Cfg = TmaCfg<CI, CP>;
    constexpr int NC = Cfg::NC;
    constexpr int RPS = Cfg::RPS;
    constexpr int NS = Cfg::NSTAGE;
    constexpr int ROWF = Cfg::ROWF;
    extern __shared__ __align__(128) float tsm[];
    float* buf = tsm;                                                   // [NS][RPS][CI][ROWF]
    uint64_t* full = reinterpret_cast<uint64_t*>(tsm + NS * Cfg::STAGE_FLOATS);
    __shared__ int s_ya[kMaxTR];
    __shared__ float s_fy[kMaxTR];

    const int H = P.H, W = P.W, h = P.h, w = P.w;
    const int tid = threadIdx.x;
    const int cb = blockIdx.x % P.ncb;
    const int k0 = blockIdx.x / P.ncb;
    const int X0 = cb * ROWF;
    const int segf = min(ROWF, W - X0);                 // floats in this column block's rows
    const uint32_t seg_bytes = (uint32_t)segf * 4u;
    const int bands = (H + P.TR - 1) / P.TR;
    const int items = P.images * bands;
    const size_t N = (size_t)H * W, n = (size_t)h * w;

    if (tid == 0) {
        for (int s = 0; s < NS; ++s) mbar_init(&full[s], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();

    // ---- producer state (thread 0): next (item, row) to stream.
    int p_item = k0, p_row = 0;
    uint64_t pol = 0;
    if (tid == 0) pol = evict_first_policy();
    auto produce = [&](int slot) {
        // issue the next stage (<= RPS rows of the current item) into `slot`
        if (p_item >= items) return;
        const int img = p_item / bands, band = p_item % bands;
        const int Yb = band * P.TR;
        const int rows_item = min(P.TR, H - Yb);
        const int nr = min(RPS, rows_item - p_row);
        mbar_expect_tx(&full[slot], (uint32_t)nr * CI * seg_bytes);
        float* dstb = buf + (size_t)slot * Cfg::STAGE_FLOATS;
        for (int r = 0; r < nr; ++r)
            for (int j = 0; j < CI; ++j)
                bulk_g2s(dstb + ((size_t)r * CI + j) * ROWF,
                         P.I + ((size_t)img * CI + j) * N + (size_t)(Yb + p_row + r) * W + X0,
                         seg_bytes, &full[slot], pol);
        p_row += nr;
        if (p_row >= rows_item) {
            p_row = 0;
            p_item += P.cpb;
        }
    };
    if (tid == 0)
        for (int s = 0; s < NS; ++s) produce(s);

    // ---- consumer: each thread owns pixels X0 + 4 tid .. + 3 of every row.
    const int xl = tid * 4;
    const bool act = xl < segf;
    const int X = X0 + xl;
    int oa[4], ob[4];
    float fx[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) src_coord(min(X + i, W - 1), w, W, oa[i], ob[i], fx[i]);

    int stage = 0;                                       // global stage counter (ring position)
    for (int item = k0; item < items; item += P.cpb) {
        const int img = item / bands, band = item % bands;
        const int Yb = band * P.TR;
        const int rows_item = min(P.TR, H - Yb);
        const float* Mb = P.M + (size_t)img * NC * n;
        float* qb = P.q + (size_t)img * CP * N + (size_t)Yb * W + X;
        // Row table of this band (R5): low-res row and vertical weight of each row.
        for (int t = tid; t < rows_item; t += 256) {
            int a, b;
            float f;
            src_coord(Yb + t, h, H, a, b, f);
            s_ya[t] = a;
            s_fy[t] = f;
        }
        __syncthreads();
        int cy = -2;
        float H0[NC][4], H1[NC][4];
        float pa[NC][4], pb[NC][4];          // raw low-res values of the prefetched row
        int py = -1;                          // low-res row held in pa/pb
        auto fetch = [&](int y) {
            const float* mr = Mb + (size_t)y * w;
#pragma unroll
            for (int m = 0; m < NC; ++m)
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    pa[m][i] = __ldg(mr + (m * (int)n + oa[i]));
                    pb[m][i] = __ldg(mr + (m * (int)n + ob[i]));
                }
            py = y;
        };
        auto lerpx = [&](float (&out)[NC][4]) {
#pragma unroll
            for (int m = 0; m < NC; ++m)
#pragma unroll
                for (int i = 0; i < 4; ++i) out[m][i] = fmaf(fx[i], pb[m][i] - pa[m][i], pa[m][i]);
        };
        auto hrow = [&](int y, float (&out)[NC][4]) {
            if (py != y) fetch(y);
            lerpx(out);
        };
        for (int r0 = 0; r0 < rows_item; r0 += RPS, ++stage) {
            const int slot = stage % NS;
            mbar_wait(&full[slot], (uint32_t)((stage / NS) & 1));
            const float* sb = buf + (size_t)slot * Cfg::STAGE_FLOATS + xl;
            const int nr = min(RPS, rows_item - r0);
#pragma unroll
            for (int r = 0; r < RPS; ++r) {
                if (r < nr) {
                    const int ya = s_ya[r0 + r];
                    const float fy = s_fy[r0 + r];
                    // ya is the same for every thread (CTA-uniform): vote -> a real branch
                    if (__any_sync(0xffffffffu, ya != cy)) {
                        if (act) {
                            const int y1 = min(ya + 1, h - 1);
                            if (ya == cy + 1) {
#pragma unroll
                                for (int m = 0; m < NC; ++m)
#pragma unroll
                                    for (int i = 0; i < 4; ++i) H0[m][i] = H1[m][i];
                            } else {
                                hrow(ya, H0);
                            }
                            hrow(y1, H1);
                            // one row ahead: the loads fly while the next ~s rows are computed
                            fetch(min(y1 + 1, h - 1));
                        }
                        cy = ya;
                    }
                    if (act) {
                        float4 iv[CI];
#pragma unroll
                        for (int j = 0; j < CI; ++j)
                            iv[j] = *reinterpret_cast<const float4*>(sb + ((size_t)r * CI + j) * ROWF);
                        float* qrow = qb + (size_t)(r0 + r) * W;
#pragma unroll
                        for (int c = 0; c < CP; ++c) {
                            const int mb = c * (CI + 1);
                            float o[4];
#pragma unroll
                            for (int i = 0; i < 4; ++i) {
                                float acc = fmaf(fy, H1[mb + CI][i] - H0[mb + CI][i], H0[mb + CI][i]);
#pragma unroll
                                for (int j = 0; j < CI; ++j) {
                                    const float a = fmaf(fy, H1[mb + j][i] - H0[mb + j][i], H0[mb + j][i]);
                                    const float v = i == 0 ? iv[j].x : (i == 1 ? iv[j].y : (i == 2 ? iv[j].z : iv[j].w));
                                    acc = fmaf(a, v, acc);
                                }
                                o[i] = acc;
                            }
                            __stcs(reinterpret_cast<float4*>(qrow + c * N), make_float4(o[0], o[1], o[2], o[3]));
                        }
                    }
                }
            }
            __syncthreads();                      // every thread is done with this slot
            if (tid == 0) {
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                produce(slot);
            }
        }
    }
}

}  // namespace fgf
