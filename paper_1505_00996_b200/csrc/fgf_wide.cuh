// fgf_wide.cuh -- K5: the whole guided filter chain for gray guidance in ONE persistent kernel
// whose per-pixel cost does not depend on the window radius.
//
//   * s = 1 (OUTQ): Algorithm 1 of the paper -- the exact guided filter:
//       mean_I, mean_p, corr_I, corr_Ip = f_mean(., r)
//       var_I, cov_Ip, a = cov_Ip / (var_I + eps), b = mean_p - a mean_I  (Eq.2-3)
//       mean_a, mean_b = f_mean(a, b)
//       q = mean_a .* I + mean_b                                    (Eq.4)
//     reading I and p once from HBM and writing q once (12 B per pixel).
//   * s > 1: steps 2-5 of Alg. 2 on the nearest samples I[y s][x s] read in place
//     (or K0's block-mean planes) for wide low-res windows r' -- mean_a, mean_b out, K4 next.
//
// Work item = (strip of TW output columns, segment of TH output rows, image); a persistent
// grid of two CTAs per SM (<= 384 threads, <= 85 registers, ~80 KB of shared memory each)
// walks the items, so one CTA's barrier / latency phases overlap the other's.  Per item the CTA streams down the rows in batches
// of G rows; every step is an O(1)-per-pixel running or prefix sum ("independent of the
// filter size"):
//
//   P0  column threads (one per statistics column, TW + 4r of them) keep fp64 running vertical
//       window sums of I, I^2, p, I p (add row y + r, subtract row y - r - 1, R1 clipping by
//       the row bounds) and snapshot them to shared memory;
//   P1  every snapshotted row becomes its fp64 prefix sum (one warp per row: each lane holds a
//       contiguous odd-length chunk in registers -- conflict-free fp64 banks -- and a warp
//       shuffle scan of the chunk totals gives the offsets);
//   P2  the horizontal window sum of a, b column j is P[j + 2r] - P[j - 1]; the coefficient
//       epilogue (fp64 var / cov, R8 clamp, fp32 quotient) writes a, b for TW + 2r columns;
//   P3  the a, b rows become fp64 prefix sums the same way;
//   P4  per output column: hb = P[t + 2r] - P[t - 1] (horizontal box of a, b), and the vertical
//       window of hb is a running fp64 sum whose subtracted rows come back from a per-CTA ring
//       of the last 2r + 1 hb rows kept in global memory (L2-resident: 148 rings); then
//       q = mean_a I + mean_b (s = 1) or the mean maps are stored (s > 1).
//
// Precision (R13, R17): products of two floats are exact in fp64; vertical sums and
// prefixes in fp64 (prefixes over <= 672 columns of sums of <= 2r+1 rows: the difference of
// two prefixes is exact to ~1e-15 relative); var / cov in fp64; quotient and b in fp32 (as the
// other engines); a, b prefixes in fp64; hb rounded to fp32 once, and the ring returns that
// same fp32 value, so the fp64 vertical sum of hb cancels exactly (no drift with the height).
//
// Nothing here is shared with oracle/ (the independent CPU reference).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "fgf_kernels.cuh"

namespace fgf {

constexpr int kWideChMax = 13;          // prefix chunk per lane: rows of <= 32 * 13 = 416 columns
constexpr int kWidePitch = 32 * kWideChMax;   // fp64 row pitch of the snapshot / a, b rows
constexpr int kWideMaxCols = 384;       // threads per CTA = statistics columns TW + 4R (rounded)
constexpr int kWideCtasPerSM = 2;

struct WideLayout {
    int NCS, NCA;          // statistics columns TW + 4R, a, b columns TW + 2R
    size_t oVA, oAB, oInvA, oInvB, oStage, oBar, total;
};

struct WideParams {
    // Sample (y, x) of image b: srcI[b*imgI + y*row + x*col]; p channel c at
    // srcP[b*imgP + c*planeP + y*row + x*col] (element type E).  In-image offsets fit in 32 bits.
    const void* srcI;
    const void* srcP;
    long long imgI, imgP;
    int planeP;
    int row, col;
    int h, w, R;           // sample-grid dims and window radius (r at s = 1, r' otherwise)
    int TW, TH;            // output columns per strip, output rows per segment
    int strips, segs, items;
    double eps;
    float k1, k0;          // written value k1 mean_a + k0 (map 0) / k1 mean (others)
    float* dst;            // maps mode: [img][2CP][h][w] fp32 (mean_a_c at 2c, mean_b_c at 2c+1)
    void* q;               // OUTQ: [img][CP][h][w] of E (s = 1: the output image itself)
    float* ring;           // [gridDim.x][2R+1][2CP][TW] fp32 ring of hb rows per CTA
    WideLayout L;
};

constexpr int kWideBulkPitch = kWideMaxCols + 8;   // floats per bulk-staged row (16 B aligned)

// STAGE: 0 = next batch's samples prefetched into registers (8/16-bit samples), 1 = by per-thread
// cp.async into shared memory (fp32, strided samples), 2 = by TMA bulk copies of whole row
// segments issued by one thread (fp32, contiguous 16-byte-aligned rows: s = 1 and K0 planes).
template <int CP, int G, int STAGE = 1>
struct WideCfg {
    static constexpr int NMAP = 2 + 2 * CP;   // I, II, p_c, Ip_c
    static constexpr int NAB = 2 * CP;        // a_c, b_c
    static constexpr int NIN = 1 + CP;        // I, p_c
    __host__ static WideLayout layout(int TW, int R) {
        WideLayout L;
        L.NCS = TW + 4 * R;
        L.NCA = TW + 2 * R;
        auto al = [](size_t x) { return (x + 15) & ~(size_t)15; };
        size_t o = 0;
        L.oVA = o; o = al(o + (size_t)G * NMAP * kWidePitch * 8);
        L.oAB = o; o = al(o + (size_t)G * NAB * kWidePitch * 8);
        L.oInvA = o; o = al(o + (size_t)kWidePitch * 8);
        L.oInvB = o; o = al(o + (size_t)kWidePitch * 4);
        // cp.async staging of the next batch's add / subtract sample rows (fp32 samples)
        L.oStage = o;
        o = al(o + (STAGE == 2 ? (size_t)G * 2 * NIN * kWideBulkPitch * 4
                               : STAGE == 1 ? (size_t)G * 2 * NIN * kWideMaxCols * 4 : 0));
        L.oBar = o; o = al(o + 16);
        L.total = o;
        return L;
    }
};

// In-place inclusive fp64 prefix sum of row[0, n) (n <= kWidePitch) by one warp: lane l owns
// the contiguous chunk [13 l, 13 l + 13) (odd length: the 16 lanes of a half-warp hit 16
// distinct fp64 banks), loaded into registers at once; a warp shuffle scan of the chunk
// totals gives the offsets.  Entries in [n, kWidePitch) are zeros that are read but never
// written.
// SPLIT = true: the chunk's own prefix is formed first, as two half-chunk chains joined by one
// add (dependent depth 7, not 13), under the latency of the shuffle scan, and the scanned
// offset is then added to every entry independently (mean-maps mode, 2 CTAs / SM: config 4
// s = 2 31.7 -> 30.0 ms); false: totals first, then one running chain (the fused s = 1 mode,
// one CTA / SM: 12.97 vs 13.14 ms with SPLIT).
template <bool SPLIT, int NR = 1>
__device__ __forceinline__ void warp_prefix_rows(double* __restrict__ row0, int stride, int n,
                                                 int lane) {
    // NR rows (row0 + k stride) scanned together: independent chains interleaved (ILP NR)
    double v[NR][kWideChMax];
#pragma unroll
    for (int k = 0; k < NR; ++k) {
        const double* r = row0 + (size_t)k * stride + lane * kWideChMax;
#pragma unroll
        for (int i = 0; i < kWideChMax; ++i) v[k][i] = r[i];
    }
    const int e = n - lane * kWideChMax;       // valid entries of this chunk
    double tot[NR], base[NR];
    if constexpr (SPLIT) {
        constexpr int H1 = (kWideChMax + 1) / 2;   // half-chunks [0, H1), [H1, 13)
#pragma unroll
        for (int i = 1; i < kWideChMax; ++i)
#pragma unroll
            for (int k = 0; k < NR; ++k)
                if (i != H1) v[k][i] += v[k][i - 1];   // two independent chains per row
#pragma unroll
        for (int i = H1; i < kWideChMax; ++i)
#pragma unroll
            for (int k = 0; k < NR; ++k) v[k][i] += v[k][H1 - 1];
#pragma unroll
        for (int k = 0; k < NR; ++k) tot[k] = v[k][kWideChMax - 1];
    } else {
#pragma unroll
        for (int k = 0; k < NR; ++k) {
            double t0 = 0.0, t1 = 0.0;             // two chains: half the dependent latency
#pragma unroll
            for (int i = 0; i < kWideChMax; i += 2) {
                t0 += v[k][i];
                if (i + 1 < kWideChMax) t1 += v[k][i + 1];
            }
            tot[k] = t0 + t1;
        }
    }
    double x[NR];
#pragma unroll
    for (int k = 0; k < NR; ++k) x[k] = tot[k];
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
#pragma unroll
        for (int k = 0; k < NR; ++k) {
            const double y = __shfl_up_sync(0xffffffffu, x[k], d);
            if (lane >= d) x[k] += y;
        }
    }
#pragma unroll
    for (int k = 0; k < NR; ++k) base[k] = x[k] - tot[k];   // exclusive scan of the totals
#pragma unroll
    for (int k = 0; k < NR; ++k) {
        double* r = row0 + (size_t)k * stride + lane * kWideChMax;
        if constexpr (SPLIT) {
#pragma unroll
            for (int i = 0; i < kWideChMax; ++i)
                if (i < e) r[i] = base[k] + v[k][i];
        } else {
            double run = base[k];
#pragma unroll
            for (int i = 0; i < kWideChMax; ++i) {
                run += v[k][i];
                if (i < e) r[i] = run;
            }
        }
    }
}

// nrows rows (row0 + rs PW) over the NW warps of the CTA: pairs of rows per warp while two
// are left for it (P2 = true), then single rows.
template <bool SPLIT, bool P2>
__device__ __forceinline__ void warp_prefix_all(double* __restrict__ row0, int nrows, int n,
                                                int warp, int NW, int lane) {
    int rs = warp;
    if constexpr (P2) {
        for (; rs + NW < nrows; rs += 2 * NW)
            warp_prefix_rows<SPLIT, 2>(row0 + (size_t)rs * kWidePitch, NW * kWidePitch, n, lane);
    }
    for (; rs < nrows; rs += NW) warp_prefix_rows<SPLIT, 1>(row0 + (size_t)rs * kWidePitch, 0, n, lane);
}

// Number of indices of [i - R, i + R] inside [0, n).
__device__ __forceinline__ int wide_count(int i, int n, int R) {
    return min(n - 1, i + R) - max(0, i - R) + 1;
}

// grid: persistent (<= items CTAs, two per SM), block NT = round32(TW + 4R) <= 384, dynamic
// smem L.total.
template <int CP, int G, bool OUTQ, typename E, int MINB = kWideCtasPerSM, bool BULK = false>
__global__ void __launch_bounds__(kWideMaxCols, MINB) wide_gray_kernel(WideParams P) {
    // fp32 samples: the next batch's rows are prefetched into shared memory (no registers held
    // while in flight) -- by TMA bulk copies of whole row segments when the rows are contiguous
    // and aligned (BULK), else by per-thread cp.async; 8/16-bit samples: into registers
    constexpr bool STAGE = sizeof(E) == 4;
    constexpr int SMODE = BULK ? 2 : (STAGE ? 1 : 0);
    static_assert(!BULK || sizeof(E) == 4, "bulk staging moves fp32 rows");
    using C = WideCfg<CP, G, SMODE>;
    constexpr int NMAP = C::NMAP, NAB = C::NAB, NIN = 1 + CP, PW = kWidePitch;
    extern __shared__ __align__(16) unsigned char smem[];
    double* __restrict__ VA = reinterpret_cast<double*>(smem + P.L.oVA);     // [G][NMAP][PW]
    double* __restrict__ AB = reinterpret_cast<double*>(smem + P.L.oAB);     // [G][NAB][PW]
    double* __restrict__ invA = reinterpret_cast<double*>(smem + P.L.oInvA); // [NCA], 0 outside
    float* __restrict__ invB = reinterpret_cast<float*>(smem + P.L.oInvB);   // [TW]
    float* __restrict__ stg = reinterpret_cast<float*>(smem + P.L.oStage);   // [G][2][NIN][384 | 392]
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem + P.L.oBar);            // BULK: rows landed
    uint32_t phase = 0;                                                      // BULK: parity
    const int NT = blockDim.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int NW = NT >> 5;
    const int h = P.h, w = P.w, R = P.R, TW = P.TW;
    const int NCS = P.L.NCS, NCA = P.L.NCA;
    const int RS = 2 * R + 1;
    const long long row = P.row;
    const double invRow = 1.0 / (double)RS;                 // interior row count

    // zero pads once: prefix rows read [n, PW) as zeros and never write them
    for (int i = tid; i < G * NMAP * PW; i += NT) VA[i] = 0.0;
    for (int i = tid; i < G * NAB * PW; i += NT) AB[i] = 0.0;
    if (BULK && tid == 0) {
        mbar_init_cta(bar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }

    // hb ring of this CTA: slot k, map m, output column t at ring[(k NAB + m) TW + t]
    float* const ring0 = P.ring + (size_t)blockIdx.x * RS * NAB * TW + tid;
    const int slotStride = NAB * TW;
    const int ringLen = RS * slotStride;              // ring offsets (floats) wrap at ringLen
    auto ldE = [](const E* p) { return ElemT<E>::load(p); };

    for (int item = blockIdx.x; item < P.items; item += gridDim.x) {
        const int strip = item % P.strips;
        const int rest = item / P.strips;
        const int seg = rest % P.segs;
        const int img = rest / P.segs;
        const int x0 = strip * TW;
        const int y0 = seg * P.TH;
        const int y1 = min(h, y0 + P.TH);                 // output rows [y0, y1)
        const int yA0 = max(0, y0 - R), yA1 = min(h, y1 + R);   // a, b rows [yA0, yA1)
        const int yEnd = y1 + R;                          // steps ya in [yA0, yEnd)

        __syncthreads();   // the previous item's P0 / P2 / P4 have read stg / invA / invB
        if (BULK) {
            // columns outside the image are never copied: they read these zeros
            for (int i = tid; i < G * 2 * NIN * kWideBulkPitch; i += NT) stg[i] = 0.0f;
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        }
        for (int j = tid; j < NCA; j += NT) {
            const int ca = x0 - R + j;
            invA[j] = (ca >= 0 && ca < w) ? 1.0 / (double)wide_count(ca, w, R) : 0.0;
        }
        for (int t = tid; t < TW; t += NT)
            invB[t] = (float)(1.0 / (double)wide_count(min(x0 + t, w - 1), w, R));

        // ---- this thread's statistics column (P0)
        const int cs = x0 - 2 * R + tid;
        const bool colS = tid < NCS;
        const bool colIn = colS && cs >= 0 && cs < w;
        const E* const colI = static_cast<const E*>(P.srcI) + img * P.imgI + (long long)(colIn ? cs : 0) * P.col;
        const E* const colP = static_cast<const E*>(P.srcP) + img * P.imgP + (long long)(colIn ? cs : 0) * P.col;
        const long long cstr = P.planeP;
        double acc[NMAP];
#pragma unroll
        for (int m = 0; m < NMAP; ++m) acc[m] = 0.0;
        if (colIn) {
            // warm-up: the window of a, b row yA0 - 1: sample rows [yA0 - 1 - R, yA0 - 1 + R]
            const int wa = max(0, yA0 - 1 - R), wb = min(h, yA0 + R);
            const E* pi = colI + wa * row;
            const E* pp = colP + wa * row;
            constexpr int WB = 8;
            for (int yy = wa; yy < wb; yy += WB) {
                float v[WB][NIN];
#pragma unroll
                for (int k = 0; k < WB; ++k) {
                    if (yy + k < wb) {
                        v[k][0] = ldE(pi + k * row);
#pragma unroll
                        for (int c = 0; c < CP; ++c) v[k][1 + c] = ldE(pp + c * cstr + k * row);
                    }
                }
#pragma unroll
                for (int k = 0; k < WB; ++k) {
                    if (yy + k < wb) {
                        const double I = (double)v[k][0];
                        acc[0] += I;
                        acc[1] = fma(I, I, acc[1]);
#pragma unroll
                        for (int c = 0; c < CP; ++c) {
                            const double pv = (double)v[k][1 + c];
                            acc[2 + c] += pv;
                            acc[2 + CP + c] = fma(I, pv, acc[2 + CP + c]);
                        }
                    }
                }
                pi += WB * row;
                pp += WB * row;
            }
        }
        // add / subtract sample rows of a batch, prefetched one batch ahead; rows that must
        // not contribute are zeros (which add exactly nothing)
        float va[STAGE ? 1 : G][NIN], vs[STAGE ? 1 : G][NIN];
        float* const stg_t = stg + tid;                   // [(g 2 + a) NIN + k] * 384
        auto stage4 = [&](int slot, const E* src, bool ok) {
            const uint32_t d = (uint32_t)__cvta_generic_to_shared(stg_t + slot * kWideMaxCols);
            asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;"
                         ::"r"(d), "l"(ok ? src : colI), "r"(ok ? 4 : 0) : "memory");
        };
        // BULK: one thread copies the batch's add / subtract sample-row segments (all planes)
        // [ca, cb) of each row into the staging rows, completion on the mbarrier (tx bytes)
        const int cs0a = (x0 - 2 * R) & ~3;                 // 16-byte-aligned segment origin
        const int bca = max(0, cs0a), bcb = min(w, (x0 - 2 * R + NCS + 3) & ~3);
        const int boff = (x0 - 2 * R) - cs0a;               // staging index of column x0 - 2R
        auto bulk_batch = [&](int ya) {
            const uint32_t nb = bcb > bca ? (uint32_t)(bcb - bca) * 4u : 0u;
            int rows = 0;
#pragma unroll
            for (int g = 0; g < G; ++g) {
                const int y = ya + g;
                rows += (y < yA1 && y + R < h) + (y < yA1 && y - R - 1 >= 0);
            }
            const uint32_t tx = nb * (uint32_t)(rows * NIN);
            const uint32_t b = smem_addr(bar);
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(tx) : "memory");
            if (nb == 0) return;
            const float* baseI = static_cast<const float*>(P.srcI) + img * P.imgI + bca;
            const float* baseP = static_cast<const float*>(P.srcP) + img * P.imgP + bca;
            auto copy = [&](int slot, const float* src) {
                const uint32_t d = smem_addr(stg + slot * kWideBulkPitch + (bca - cs0a));
                asm volatile(
                    "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                    ::"r"(d), "l"(src), "r"(nb), "r"(b) : "memory");
            };
#pragma unroll
            for (int g = 0; g < G; ++g) {
                const int y = ya + g;
                if (y < yA1 && y + R < h) {
                    copy((g * 2 + 0) * NIN, baseI + (long long)(y + R) * row);
#pragma unroll
                    for (int c = 0; c < CP; ++c)
                        copy((g * 2 + 0) * NIN + 1 + c, baseP + c * cstr + (long long)(y + R) * row);
                }
                if (y < yA1 && y - R - 1 >= 0) {
                    copy((g * 2 + 1) * NIN, baseI + (long long)(y - R - 1) * row);
#pragma unroll
                    for (int c = 0; c < CP; ++c)
                        copy((g * 2 + 1) * NIN + 1 + c, baseP + c * cstr + (long long)(y - R - 1) * row);
                }
            }
        };
        auto load_batch = [&](int ya) {
            const E* ai = colI + (ya + R) * row;
            const E* ap = colP + (ya + R) * row;
            const E* si = colI + (ya - R - 1) * row;
            const E* sp = colP + (ya - R - 1) * row;
            const bool full = colIn && ya + G <= yA1 && ya - R - 1 >= 0 && ya + G - 1 + R < h;
#pragma unroll
            for (int g = 0; g < G; ++g) {
                const int y = ya + g;
                const bool oka = full || (colIn && y < yA1 && y + R < h);
                const bool oks = full || (colIn && y < yA1 && y - R - 1 >= 0);
                if constexpr (STAGE) {
                    stage4((g * 2 + 0) * NIN, ai, oka);
                    stage4((g * 2 + 1) * NIN, si, oks);
#pragma unroll
                    for (int c = 0; c < CP; ++c) {
                        stage4((g * 2 + 0) * NIN + 1 + c, ap + c * cstr, oka);
                        stage4((g * 2 + 1) * NIN + 1 + c, sp + c * cstr, oks);
                    }
                    ai += row; ap += row; si += row; sp += row;
                } else {
                    va[STAGE ? 0 : g][0] = oka ? ldE(ai + g * row) : 0.0f;
                    vs[STAGE ? 0 : g][0] = oks ? ldE(si + g * row) : 0.0f;
#pragma unroll
                    for (int c = 0; c < CP; ++c) {
                        va[STAGE ? 0 : g][1 + c] = oka ? ldE(ap + c * cstr + g * row) : 0.0f;
                        vs[STAGE ? 0 : g][1 + c] = oks ? ldE(sp + c * cstr + g * row) : 0.0f;
                    }
                }
            }
            if constexpr (STAGE) asm volatile("cp.async.commit_group;" ::: "memory");
        };

        // ---- this thread's output column (P4)
        const int xo = x0 + tid;
        const bool colO = tid < TW && xo < w;
        const E* const Iq = static_cast<const E*>(P.srcI) + img * P.imgI + xo;   // OUTQ: s = 1
        double accB[NAB];
#pragma unroll
        for (int m = 0; m < NAB; ++m) accB[m] = 0.0;
        int rslot = 0;                                     // ring offset of step ya
        double* const va_t = VA + tid;                     // P0 snapshots of this column
        const double* const pa_t = VA + tid;               // P2: window ends tid - 1, tid + 2R
        double* const ab_t = AB + tid;                     // P2: a, b of column tid
        const double* const pb_t = AB + tid;               // P4: window ends tid - 1, tid + 2R
        const int R2 = 2 * R;

        if (BULK) {
            __syncthreads();                                // the zeroed staging rows are visible
            if (tid == 0) bulk_batch(yA0);
        } else {
            load_batch(yA0);
        }
        for (int ya = yA0; ya < yEnd; ya += G) {
            const int nA = max(0, min(G, yA1 - ya));       // a, b rows of this batch
            const int nS = min(G, yEnd - ya);              // steps of this batch
            // ---- P0: vertical windows of a, b rows [ya, ya + nA), snapshots
            if (BULK) {
                if (nA > 0) {
                    mbar_wait_parity(bar, phase);
                    phase ^= 1u;
                }
            } else if constexpr (STAGE) {
                asm volatile("cp.async.wait_group 0;" ::: "memory");
            }
            if (colS) {
#pragma unroll
                for (int g = 0; g < G; ++g) {
                    if (g < nA) {
                        float xa[NIN], xs[NIN];
                        if (BULK) {
                            const int y = ya + g;
                            const bool oka = colIn && y + R < h, oks = colIn && y - R - 1 >= 0;
                            const float* bs = stg + boff + tid;
#pragma unroll
                            for (int k = 0; k < NIN; ++k) {
                                xa[k] = oka ? bs[((g * 2 + 0) * NIN + k) * kWideBulkPitch] : 0.0f;
                                xs[k] = oks ? bs[((g * 2 + 1) * NIN + k) * kWideBulkPitch] : 0.0f;
                            }
                        } else {
#pragma unroll
                            for (int k = 0; k < NIN; ++k) {
                                xa[k] = STAGE ? stg_t[((g * 2 + 0) * NIN + k) * kWideMaxCols] : va[STAGE ? 0 : g][k];
                                xs[k] = STAGE ? stg_t[((g * 2 + 1) * NIN + k) * kWideMaxCols] : vs[STAGE ? 0 : g][k];
                            }
                        }
                        const double Ia = (double)xa[0], Is = (double)xs[0];
                        acc[0] += Ia - Is;
                        acc[1] += fma(Ia, Ia, -(Is * Is));
#pragma unroll
                        for (int c = 0; c < CP; ++c) {
                            const double pa = (double)xa[1 + c], ps = (double)xs[1 + c];
                            acc[2 + c] += pa - ps;
                            acc[2 + CP + c] += fma(Ia, pa, -(Is * ps));
                        }
#pragma unroll
                        for (int m = 0; m < NMAP; ++m) va_t[(g * NMAP + m) * PW] = acc[m];
                    }
                }
            }
            if (!BULK && ya + G < yA1) load_batch(ya + G);
            if (BULK) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // reads before the next copies
            // ring rows leaving the vertical windows of this batch's steps, and (s = 1) the
            // guidance row of each output: issued now, used in P4
            float old[G][NAB];
            float Io[OUTQ ? G : 1];
            // interior batches (warp-uniform): every step removes a ring row and emits an output
            const bool fastS = nS == G && ya - RS >= yA0;
            const bool fastO = nS == G && ya - R >= y0 && ya + G - 1 - R < y1;
            if (colO) {
                int ro = rslot;
                const E* ip = Iq + (ya - R) * row;
#pragma unroll
                for (int g = 0; g < G; ++g) {
                    const int yy = ya + g;
                    const bool sub = fastS || (g < nS && yy - RS >= yA0);   // row yy - 2R - 1 was added
#pragma unroll
                    for (int m = 0; m < NAB; ++m) old[g][m] = sub ? ring0[ro + m * TW] : 0.0f;
                    if (OUTQ) {
                        const int yb = yy - R;
                        Io[OUTQ ? g : 0] = (fastO || (g < nS && yb >= y0 && yb < y1)) ? ldE(ip) : 0.0f;
                        ip += row;
                    }
                    ro += slotStride;
                    ro = ro == ringLen ? 0 : ro;
                }
            }
            __syncthreads();
            if (BULK && tid == 0 && ya + G < yA1) bulk_batch(ya + G);   // in flight under P1-P4
            // ---- P1: prefix sums of the snapshotted rows
            warp_prefix_all<!OUTQ, OUTQ>(VA, nA * NMAP, NCS, warp, NW, lane);
            __syncthreads();
            // ---- P2: window sums, coefficient epilogue -> a, b (fp64 rows for P3)
            if (tid < NCA) {
                const double ix = invA[tid];
                const bool first = tid == 0;
#pragma unroll
                for (int g = 0; g < G; ++g) {
                    if (g < nA) {
                        const int yy = ya + g;
                        const double iy = (yy - R >= 0 && yy + R < h)
                                              ? invRow : 1.0 / (double)wide_count(yy, h, R);
                        const double inv = ix * iy;           // 0 outside the image -> a = b = 0
                        double S[NMAP];
#pragma unroll
                        for (int m = 0; m < NMAP; ++m) {
                            const double* q = pa_t + (g * NMAP + m) * PW;
                            S[m] = q[R2] - (first ? 0.0 : q[-1]);
                        }
                        const double mI = S[0] * inv;
                        double var = fma(-mI, mI, S[1] * inv);     // var_I (P:58 / P:78)
                        var = var < 0.0 ? 0.0 : var;               // R8
                        float rden;                                // 1 / (var + eps), ~1 ulp
                        asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(rden) : "f"((float)(var + P.eps)));
                        const float mIf = (float)mI;
#pragma unroll
                        for (int c = 0; c < CP; ++c) {
                            const double mp = S[2 + c] * inv;
                            const double cov = fma(-mI, mp, S[2 + CP + c] * inv);   // cov_Ip
                            const float a = (float)cov * rden;                    // Eq.2
                            ab_t[(g * NAB + 2 * c) * PW] = (double)a;
                            ab_t[(g * NAB + 2 * c + 1) * PW] = (double)fmaf(-a, mIf, (float)mp);   // Eq.3
                        }
                    }
                }
            }
            __syncthreads();
            // ---- P3: prefix sums of the a, b rows
            warp_prefix_all<!OUTQ, OUTQ>(AB, nA * NAB, NCA, warp, NW, lane);
            __syncthreads();
            // ---- P4: horizontal box of a, b, vertical running window through the ring, output
            if (colO) {
                const float ixB = invB[tid];
                const float ixR = ixB * (float)invRow;
                const bool first = tid == 0;
                const bool fastA = nA == G;
                int ro = rslot;
                E* qrow = OUTQ ? static_cast<E*>(P.q) + (long long)img * CP * h * w + (long long)(ya - R) * w + xo
                               : nullptr;
#pragma unroll
                for (int g = 0; g < G; ++g) {
                    if (fastO || g < nS) {
                        if (fastA || g < nA) {
#pragma unroll
                            for (int m = 0; m < NAB; ++m) {
                                const double* q = pb_t + (g * NAB + m) * PW;
                                const float hb = (float)(q[R2] - (first ? 0.0 : q[-1]));
                                ring0[ro + m * TW] = hb;
                                accB[m] += (double)hb;
                            }
                        }
#pragma unroll
                        for (int m = 0; m < NAB; ++m) accB[m] -= (double)old[g][m];
                        const int yb = ya + g - R;
                        if (fastO || (yb >= y0 && yb < y1)) {
                            const float inv = (yb - R >= 0 && yb + R < h)
                                                  ? ixR : ixB / (float)wide_count(yb, h, R);
                            if (OUTQ) {
                                const float I = Io[OUTQ ? g : 0];
                                E* qo = qrow + (long long)g * w;
#pragma unroll
                                for (int c = 0; c < CP; ++c) {
                                    const float ma = fmaf(P.k1, (float)accB[2 * c] * inv,
                                                          c == 0 ? P.k0 : 0.0f);
                                    const float mb = P.k1 * ((float)accB[2 * c + 1] * inv);
                                    const float qv = fmaf(ma, I, mb);           // Eq.4
                                    const unsigned bits = ElemT<E>::bits(qv);
                                    E* qc = qo + (long long)c * h * w;
                                    if (sizeof(E) == 4) __stcs(reinterpret_cast<float*>(qc), __uint_as_float(bits));
                                    else if (sizeof(E) == 2) __stcs(reinterpret_cast<unsigned short*>(qc), (unsigned short)bits);
                                    else *reinterpret_cast<unsigned char*>(qc) = (unsigned char)bits;
                                }
                            } else {
                                float* d = P.dst + ((size_t)img * NAB * h + yb) * w + xo;
#pragma unroll
                                for (int m = 0; m < NAB; ++m)
                                    d[(size_t)m * h * w] = fmaf(P.k1, (float)accB[m] * inv, m == 0 ? P.k0 : 0.0f);
                            }
                        }
                    }
                    ro += slotStride;
                    ro = ro == ringLen ? 0 : ro;
                }
            }
            // ring offset of the next batch's first step
            rslot += G * slotStride;
            rslot = rslot >= ringLen ? rslot - ringLen : rslot;
        }
    }
}

}  // namespace fgf
