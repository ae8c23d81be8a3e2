// fgf_lowres.cuh -- K13: the whole low-resolution chain of Alg. 2 for gray
// guidance in ONE kernel.
//
//   step 1  I' = f_sub(I, s), p' = f_sub(p, s): the samples are read straight from
//                      the source through (row, col) strides -- the full-resolution image at
//                      the nearest sample sites I[y s][x s] (R3), the image itself at
//                      s = 1, or K0's compact block-mean planes (R4);
//   steps 2-4 (Eq.2-3)  mean_I, corr_I, mean_p, corr_Ip (box of radius r', R1),
//                      var_I, cov_Ip, a = cov_Ip / (var_I + eps), b = mean_p - a mean_I;
//   step 5  mean_a = f_mean(a), mean_b = f_mean(b) -> the only HBM write.
//
// A CTA owns a strip of TW output columns and a segment of TH output rows.  Stage A computes
// a, b on the strip widened by r' (TW + 2r' columns) and the segment widened by r' rows,
// which needs statistics over TW + 4r' sample columns; stage B boxes a, b into the outputs.
// Both stages are the O(1)-per-pixel running-sum box of P:16: one thread per column keeps
// fp64 vertical window sums in registers (add row y + r', subtract row y - r'), the sums of
// G rows are snapshot to shared memory, and threads slide horizontal windows along runs of
// K (odd: conflict-free fp64 banks) columns.  Stage B lags stage A by r' rows; a, b live in
// a shared-memory ring of 2r' + G rows (fp32, as stored by the unfused path), the raw samples
// in a per-thread ring of 2r' + 1 rows, so every sample is read from memory exactly once and
// nothing but mean_a, mean_b ever reaches HBM.  Window clipping: columns / rows outside the
// image contribute zeros and the divisor is the in-bounds count (R1).
//
// Precision (R13): fp64 statistics box sums (products of two floats are exact in
// fp64), fp64 var_I / cov_Ip, fp32 quotient and b (as the unfused path), fp32 a, b storage and
// fp32 box sums of a, b (stage B; R17: |a| <= sqrt(var_p)/(2 sqrt(eps)), so the
// fp32 sums add errors of the same order as the fp32 storage of a, b itself).
//
// Nothing here is shared with oracle/ (the independent CPU reference).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace fgf {

// Shared-memory carve-up of K13 (bytes), computed on the host by LowresCfg::layout and passed
// in the parameters.
struct LowresLayout {
    int NT, NCA, NCS, nrA, nrB, PA, PB, VPA, VPB, RBA, RBI, THA, THB;
    int RVB, ROS, RAB;     // row pitches (floats) of VsB, Os and the a, b ring slots
    size_t oVsA, oVsB, oInvxA, oInvxB, oInvyA, oInvyB, oABr, oINr, oOs, total;
};

struct LowresParams {
    // Sample (y, x) of image b: srcI[b*imgI + y*row + x*col]; p channel c at
    // srcP[b*imgP + c*planeP + y*row + x*col].  In-image offsets fit in 32 bits (validated).
    const void* srcI;      // element type E of the kernel (float, __half, __nv_bfloat16)
    const void* srcP;
    long long imgI, imgP;
    int planeP;
    int row, col;
    float* dst;            // [img][2CP][h][w]: mean_a_c at 2c, mean_b_c at 2c+1
    int h, w, R;
    int TW, TH;            // output columns per strip, output rows per segment
    double eps;
    float k1, k0;          // written maps: k1 mean_a + k0 (map 0), k1 mean (others); 1, 0 = plain
    int bulk_out;          // 1: the staged output rows go out as TMA bulk copies (host-checked:
                           // w, TW and the Os pitches multiples of 4 floats, dst 16-byte aligned)
    LowresLayout L;        // LowresCfg<...>::layout(blockDim.x, TW, TH, R), set by the host
};

// Bulk shared -> global copy of `bytes` (multiple of 16, both addresses 16-byte aligned) by
// the async proxy; completion tracked per issuing thread by bulk groups.
__device__ __forceinline__ void lr_bulk_store(float* gdst, const float* ssrc, unsigned bytes) {
    const unsigned s = (unsigned)__cvta_generic_to_shared(ssrc);
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;"
                 ::"l"(gdst), "r"(s), "r"(bytes) : "memory");
}

template <int CP, int G, int KA, int KB, bool RING = true>
struct LowresCfg {
    static constexpr int NIN = 1 + CP;          // I', p'_c
    static constexpr int NMAP = 2 + 2 * CP;     // I', I'I', p'_c, I'p'_c
    static constexpr int NAB = 2 * CP;          // a_c, b_c
    // Shared-memory carve-up (bytes); identical on host and device.  Every horizontal run
    // may read / write past the last valid column: the pitches are padded so those accesses
    // stay inside zero-initialised (read) or scratch (write) padding.
    using Layout = LowresLayout;
    __host__ __device__ static size_t al16(size_t x) { return (x + 15) & ~(size_t)15; }
    __host__ __device__ static Layout layout(int NT, int TW, int TH, int R) {
        Layout L;
        L.NT = NT;
        L.NCA = TW + 2 * R;                      // a, b columns
        L.NCS = TW + 4 * R;                      // sample / statistics columns
        L.nrA = (L.NCA + KA - 1) / KA;           // stage-A runs per row
        L.nrB = (TW + KB - 1) / KB;              // stage-B runs per row
        L.PA = L.nrA * KA;                       // padded a, b row (ABr, invxA)
        L.PB = L.nrB * KB;                       // padded output row (Os, invxB)
        L.VPA = L.PA + 2 * R + 1;                // sums pitch: every run's reads in bounds
        if (L.VPA < NT) L.VPA = NT;
        L.VPB = L.PB + 2 * R + 1;
        if (L.VPB < L.PA) L.VPB = L.PA;
        L.RBA = 2 * R + G + 1;                   // a, b rows [yb - R - 1, yA) live at once
        L.RBI = 2 * R + 2;                       // sample rows [ya - R - 1, ya + R]
        L.THA = TH + 2 * R + 2;                  // a, b rows of a segment (1 / count table)
        L.THB = TH;
        // Row pitches p = q (mod 32) words, q = the runs of a row times the run length: the
        // run threads of one warp span consecutive rows, and with this pitch lane l of the
        // warp addresses word 9 l + const (mod 32) -- distinct banks (K odd).
        auto pitch = [](int base, int runs, int K) {
            const int want = (runs * K) & 31;
            return base + ((want - base) & 31);
        };
        L.RVB = pitch(NAB * L.VPB, L.nrB, KB);
        L.ROS = pitch(NAB * L.PB, L.nrB, KB);
        L.RAB = pitch(NAB * L.PA, L.nrA, KA);
        size_t o = 0;
        L.oVsA = o; o = al16(o + (size_t)G * NMAP * L.VPA * 8);
        L.oVsB = o; o = al16(o + (size_t)G * L.RVB * 4);
        L.oInvxA = o; o = al16(o + (size_t)L.PA * 8);
        L.oInvxB = o; o = al16(o + (size_t)L.PB * 4);
        L.oInvyA = o; o = al16(o + (size_t)L.THA * 8);
        L.oInvyB = o; o = al16(o + (size_t)L.THB * 4);
        L.oABr = o; o = al16(o + (size_t)L.RBA * L.RAB * 4);
        L.oINr = o; o = al16(o + (RING ? (size_t)L.RBI * NIN * NT * 4 : 0));
        L.oOs = o; o = al16(o + (size_t)G * L.ROS * 4);
        L.total = o;
        return L;
    }
};

// 1 / (number of in-bounds indices of the window [i - R, i + R] in [0, n)).
__device__ __forceinline__ double inv_count(int i, int n, int R) {
    return 1.0 / (double)(min(n - 1, i + R) - max(0, i - R) + 1);
}

// grid (strips, segments, images), block NT (>= TW + 4R, multiple of 32), dynamic smem
// LowresCfg::layout(...).total.
// RING = false: no sample ring; the subtracted row is re-read from global memory (L2) and
// prefetched together with the added row.  MAXT / MINB: launch bounds.
//
// Schedule: two barrier intervals per batch of G rows.
//   X (column threads):  stage-B column phase of the batch of outputs whose a, b windows are
//                        complete, then the stage-A column phase of the next G a, b rows;
//   Y (run threads):     stage-A horizontal phase + epilogue of those a, b rows on threads
//                        [0, TA), and concurrently the stage-B horizontal phase of the outputs
//                        on threads [TA, TA + TB); then the staged outputs are stored.
template <int CP, int G, int KA, int KB, bool RING = true, int MAXT = 512, int MINB = 1,
          typename E = float>
__global__ void __launch_bounds__(MAXT, MINB) lowres_gray_kernel(LowresParams P) {
    using C = LowresCfg<CP, G, KA, KB, RING>;
    constexpr int NIN = C::NIN, NMAP = C::NMAP, NAB = C::NAB;
    extern __shared__ __align__(16) unsigned char smem[];
    // a programmatic dependent (K4 launched with programmatic stream serialisation) may start
    // its map-independent prologue once every CTA of this grid is running; it waits for this
    // grid's completion (griddepcontrol.wait) before reading the maps.  No-op otherwise.
    asm volatile("griddepcontrol.launch_dependents;");
    const int NT = blockDim.x, tid = threadIdx.x;
    const int h = P.h, w = P.w, R = P.R, TW = P.TW;
    const LowresLayout& L = P.L;
    double* VsA = reinterpret_cast<double*>(smem + L.oVsA);     // [G][NMAP][VPA]
    float* VsB = reinterpret_cast<float*>(smem + L.oVsB);       // [G] (pitch RVB) [NAB][VPB]
    double* invxA = reinterpret_cast<double*>(smem + L.oInvxA); // [PA], 0 = outside the image
    float* invxB = reinterpret_cast<float*>(smem + L.oInvxB);   // [PB]
    double* invyA = reinterpret_cast<double*>(smem + L.oInvyA); // [THA] per a, b row - yA0
    float* invyB = reinterpret_cast<float*>(smem + L.oInvyB);   // [THB] per output row - y0
    float* ABr = reinterpret_cast<float*>(smem + L.oABr);       // [RBA] (pitch RAB) [NAB][PA]
    float* INr = reinterpret_cast<float*>(smem + L.oINr);       // [RBI][NIN][NT]
    float* Os = reinterpret_cast<float*>(smem + L.oOs);         // [G] (pitch ROS) [NAB][PB]

    const int img = blockIdx.z;
    const int x0 = blockIdx.x * TW;
    const int y0 = blockIdx.y * P.TH;
    const int yB1 = min(h, y0 + P.TH);            // outputs [y0, yB1)
    // a, b rows [yA0, yA1): the output windows need [y0 - R, yB1 + R); one more row on top
    // because stage B's first step removes row y0 - R - 1 from its running window
    const int yA0 = max(0, y0 - R - 1);
    const int yA1 = min(h, yB1 + R);
    const int VPA = L.VPA, VPB = L.VPB, PA = L.PA, PB = L.PB, RBA = L.RBA, RBI = L.RBI;

    // ---- tables and zero pads (the zeros make out-of-image columns contribute nothing
    // and make a = b = 0 there: inv = 0 turns every mean into 0)
    for (int i = tid; i < G * NMAP * VPA; i += NT) VsA[i] = 0.0;
    for (int i = tid; i < G * L.RVB; i += NT) VsB[i] = 0.0f;
    for (int j = tid; j < PA; j += NT) {
        const int ca = x0 - R + j;
        invxA[j] = (j < L.NCA && ca >= 0 && ca < w) ? inv_count(ca, w, R) : 0.0;
    }
    for (int k = tid; k < PB; k += NT) invxB[k] = (float)inv_count(min(x0 + k, w - 1), w, R);
    for (int t = tid; t < yA1 - yA0; t += NT) invyA[t] = inv_count(yA0 + t, h, R);
    for (int t = tid; t < yB1 - y0; t += NT) invyB[t] = (float)inv_count(y0 + t, h, R);

    // ---- this thread's sample column (stage A column phase)
    const int cs = x0 - 2 * R + tid;
    const bool colS = tid < L.NCS;                // owns a statistics column (maybe outside)
    const bool colA = colS && cs >= 0 && cs < w;  // ... inside the image
    const int offc = (colA ? cs : 0) * P.col;
    const E* bI = static_cast<const E*>(P.srcI) + img * P.imgI + offc;
    const E* bP = static_cast<const E*>(P.srcP) + img * P.imgP + offc;
    const int row = P.row, planeP = P.planeP;
    const long long dP = bP - bI;
    auto ld = [](const E* q) { return ElemT<E>::load(q); };
    auto load = [&](int y, float* v) {
        const E* pi = bI + (long long)y * row;
        v[0] = ld(pi);
#pragma unroll
        for (int c = 0; c < CP; ++c) v[1 + c] = ld(pi + dP + c * planeP);
    };
    // add (sub = false) or remove one sample row: [I, II, p_c, Ip_c], exact products in fp64
    auto accum = [&](double* acc, const float* v, bool sub) {
        const double I = (double)v[0];
        acc[0] = sub ? acc[0] - I : acc[0] + I;
        acc[1] = sub ? fma(-I, I, acc[1]) : fma(I, I, acc[1]);
#pragma unroll
        for (int c = 0; c < CP; ++c) {
            const double p = (double)v[1 + c];
            acc[2 + c] = sub ? acc[2 + c] - p : acc[2 + c] + p;
            acc[2 + CP + c] = sub ? fma(-I, p, acc[2 + CP + c]) : fma(I, p, acc[2 + CP + c]);
        }
    };
    const int ringStride = NIN * NT;              // floats between sample-ring slots
    float* inr = INr + tid;                       // slot s, input k at inr[s*ringStride + k*NT]

    double accA[NMAP];
#pragma unroll
    for (int m = 0; m < NMAP; ++m) accA[m] = 0.0;
    // The window of a, b row ya moves down by one row: add sample row ya + R, remove row
    // ya - R - 1.  Ring slots: row ya + R in slot (ya + R) mod RBI, row ya - R - 1 in the next
    // slot (RBI = 2R + 2).
    int sAdd = (yA0 + R) % RBI;
    if (colA) {
        // warm-up: the window of row yA0 - 1, rows [yA0 - R - 1, yA0 + R - 1] clipped
        const int wa = max(0, yA0 - R - 1), wb = min(h, yA0 + R);
        constexpr int WB = 8;                     // rows whose loads are in flight together
        for (int y0w = wa; y0w < wb; y0w += WB) {
            float v[WB][NIN];
#pragma unroll
            for (int k = 0; k < WB; ++k)
                if (y0w + k < wb) load(y0w + k, v[k]);
#pragma unroll
            for (int k = 0; k < WB; ++k) {
                const int y = y0w + k;
                if (y < wb) {
                    if (RING) {
                        int sl = sAdd + (y - yA0 - R);
                        if (sl < 0) sl += RBI;
#pragma unroll
                        for (int c = 0; c < NIN; ++c) inr[sl * ringStride + c * NT] = v[k][c];
                    }
                    accum(accA, v[k], false);
                }
            }
        }
    }
    // prefetch of the add rows (and without the ring, the subtract rows) of a batch
    float nv[G][NIN];
    float sv[RING ? 1 : G][NIN];
    auto load_batch = [&](int ya) {
        if (!colA) return;
        const int ng = min(yA1 - ya, h - (ya + R));   // add rows that exist
        const E* pi = bI + (long long)(ya + R) * row;
        if (ng >= G) {
#pragma unroll
            for (int g = 0; g < G; ++g) {
                nv[g][0] = ld(pi);
#pragma unroll
                for (int c = 0; c < CP; ++c) nv[g][1 + c] = ld(pi + dP + c * planeP);
                pi += row;
            }
        } else {
#pragma unroll
            for (int g = 0; g < G; ++g) {
                if (g < ng) {
                    nv[g][0] = ld(pi);
#pragma unroll
                    for (int c = 0; c < CP; ++c) nv[g][1 + c] = ld(pi + dP + c * planeP);
                }
                pi += row;
            }
        }
        if (!RING) {
            const int g0 = max(0, R + 1 - ya);             // subtract rows ya + g - R - 1 >= 0
            const int g1 = min(G, yA1 - ya);
            const E* ps = bI + (long long)(ya - R - 1) * row;
            if (g0 == 0 && g1 == G) {
#pragma unroll
                for (int g = 0; g < (RING ? 1 : G); ++g) {
                    sv[g][0] = ld(ps);
#pragma unroll
                    for (int c = 0; c < CP; ++c) sv[g][1 + c] = ld(ps + dP + c * planeP);
                    ps += row;
                }
            } else {
#pragma unroll
                for (int g = 0; g < (RING ? 1 : G); ++g) {
                    if (g >= g0 && g < g1) {
                        sv[g][0] = ld(ps);
#pragma unroll
                        for (int c = 0; c < CP; ++c) sv[g][1 + c] = ld(ps + dP + c * planeP);
                    }
                    ps += row;
                }
            }
        }
    };
    // one row step: acc += f(add row) - f(sub row), as one difference per map (short chains)
    auto step = [&](const float* va, const float* vs, bool hasA, bool hasS) {
        const double Ia = hasA ? (double)va[0] : 0.0, Is = hasS ? (double)vs[0] : 0.0;
        accA[0] += Ia - Is;
        accA[1] += fma(Ia, Ia, -(Is * Is));
#pragma unroll
        for (int c = 0; c < CP; ++c) {
            const double pa = hasA ? (double)va[1 + c] : 0.0, ps = hasS ? (double)vs[1 + c] : 0.0;
            accA[2 + c] += pa - ps;
            accA[2 + CP + c] += fma(Ia, pa, -(Is * ps));
        }
    };
    // stage-A column phase: vertical sums of a, b rows [ya0, ya0 + nA) -> VsA.  Columns
    // outside the image keep the zeros written at the start.
    auto column_A = [&](int ya0, int nA) {
        if (!colA) return;
        double* vcol = VsA + tid;
        if (!RING && nA == G && ya0 - R - 1 >= 0 && ya0 + G - 1 + R < h) {
            // interior batch: every add and subtract row exists -- straight-line code
#pragma unroll
            for (int g = 0; g < G; ++g) {
                step(nv[g], sv[RING ? 0 : g], true, true);
                double* v = vcol + g * NMAP * VPA;
#pragma unroll
                for (int m = 0; m < NMAP; ++m) {
                    *v = accA[m];
                    v += VPA;
                }
            }
            return;
        }
        int s = sAdd;
        const bool full = false;
#pragma unroll
        for (int g = 0; g < G; ++g) {
            if (full || g < nA) {
                const int ya = ya0 + g;
                const int ss = (s + 1 == RBI) ? 0 : s + 1;
                const bool hasA = full || ya + R < h, hasS = full || ya - R - 1 >= 0;
                float vsub[NIN];
                if (RING) {
                    if (hasA) {
                        float* slot = inr + s * ringStride;
#pragma unroll
                        for (int k = 0; k < NIN; ++k) slot[k * NT] = nv[g][k];
                    }
                    if (hasS) {
                        const float* slot = inr + ss * ringStride;
#pragma unroll
                        for (int k = 0; k < NIN; ++k) vsub[k] = slot[k * NT];
                    }
                }
                step(nv[g], RING ? vsub : sv[RING ? 0 : g], hasA, hasS);
#pragma unroll
                for (int m = 0; m < NMAP; ++m) vcol[(g * NMAP + m) * VPA] = accA[m];
                s = ss;
            }
        }
        sAdd = s;
    };

    // stage-B column state: a, b column j = tid (local), ca = x0 - R + j
    const bool colB = tid < L.NCA;
    const bool colBv = colB && x0 - R + tid >= 0 && x0 - R + tid < w;   // inside the image
    float accB[NAB];
#pragma unroll
    for (int m = 0; m < NAB; ++m) accB[m] = 0.0f;

    // horizontal tasks: q < TA -> stage A (row gA, run jA0), TA <= q < TA + TB -> stage B
    const int TA = G * L.nrA, TB = G * L.nrB;
    const int qB = tid - TA;
    const int gA = tid / L.nrA, jA0 = (tid - gA * L.nrA) * KA;
    const int gB = qB / L.nrB, kB0 = (qB - gB * L.nrB) * KB;
    const bool runA = tid < TA, runB = qB >= 0 && qB < TB;
    const double* hvA = VsA + (size_t)gA * NMAP * VPA + jA0;
    const float* hvB = VsB + (size_t)(runB ? gB : 0) * L.RVB + (runB ? kB0 : 0);

    const size_t n = (size_t)h * w;
    float* dstimg = P.dst + (size_t)img * NAB * n;

    int yA = yA0;                                 // first a, b row of the batch in VsA
    int sA = yA0 % RBA;                           // ring slot of a, b row yA
    int nA = max(0, min(G, yA1 - yA));            // a, b rows in VsA
    int yb = y0;                                  // next output row
    int hbY = 0, hbN = 0;                         // outputs whose vertical sums are in VsB

    load_batch(yA);
    column_A(yA, nA);
    if (nA > 0) load_batch(yA + nA);
    __syncthreads();
    for (;;) {
        // ================= Y: horizontal phases
        if (runA && gA < nA) {
            const int ya = yA + gA;
            const double invy = invyA[ya - yA0];
            int sl = sA + gA;
            if (sl >= RBA) sl -= RBA;
            float* ab = ABr + (size_t)sl * L.RAB + jA0;
            const double* ix = invxA + jA0;
            const double* vw = hvA + 2 * R + 1;
            double S[NMAP];
#pragma unroll
            for (int m = 0; m < NMAP; ++m) S[m] = 0.0;
#pragma unroll 4
            for (int k = 0; k <= 2 * R; ++k)
#pragma unroll
                for (int m = 0; m < NMAP; ++m) S[m] += hvA[m * VPA + k];
#pragma unroll
            for (int i = 0; i < KA; ++i) {
                const double inv = ix[i] * invy;           // 0 outside the image -> a = b = 0
                const double mI = S[0] * inv;
                double var = fma(-mI, mI, S[1] * inv);     // var_I
                var = var < 0.0 ? 0.0 : var;               // R8
                float rden;                                // 1 / (var + eps), ~1 ulp
                asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(rden) : "f"((float)(var + P.eps)));
                const float mIf = (float)mI;
#pragma unroll
                for (int c = 0; c < CP; ++c) {
                    const double mp = S[2 + c] * inv;
                    const double cov = fma(-mI, mp, S[2 + CP + c] * inv);   // cov_Ip
                    const float a = (float)cov * rden;                    // Eq.2 / P:80
                    ab[(2 * c) * PA + i] = a;
                    ab[(2 * c + 1) * PA + i] = fmaf(-a, mIf, (float)mp);  // Eq.3 / P:81
                }
                if (i + 1 < KA) {
#pragma unroll
                    for (int m = 0; m < NMAP; ++m) S[m] += vw[m * VPA + i] - hvA[m * VPA + i];
                }
            }
        }
        if (runB && gB < hbN) {
            const float invy = invyB[hbY + gB - y0];
            const float* ix = invxB + kB0;
            const float* vw = hvB + 2 * R + 1;
            float S[NAB];
#pragma unroll
            for (int m = 0; m < NAB; ++m) S[m] = 0.0f;
#pragma unroll 4
            for (int k = 0; k <= 2 * R; ++k)
#pragma unroll
                for (int m = 0; m < NAB; ++m) S[m] += hvB[m * VPB + k];
            float* o = Os + (size_t)gB * L.ROS + kB0;
#pragma unroll
            for (int i = 0; i < KB; ++i) {
                const float inv = ix[i] * invy;
#pragma unroll
                for (int m = 0; m < NAB; ++m) o[m * PB + i] = fmaf(P.k1, S[m] * inv, m == 0 ? P.k0 : 0.0f);
                if (i + 1 < KB) {
#pragma unroll
                    for (int m = 0; m < NAB; ++m) S[m] += vw[m * VPB + i] - hvB[m * VPB + i];
                }
            }
        }
        if (P.bulk_out) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // Os -> async proxy
        __syncthreads();
        // store of the outputs staged in Os: one TMA bulk copy per row and map (issued by one
        // thread; Os is not rewritten before the copies have read it, see the end of X), or
        // coalesced per-thread stores
        if (P.bulk_out) {
            if (tid == 0 && hbN > 0) {
                const unsigned bytes = (unsigned)min(TW, w - x0) * 4u;
                for (int g = 0; g < hbN; ++g) {
#pragma unroll
                    for (int m = 0; m < NAB; ++m)
                        lr_bulk_store(dstimg + (size_t)m * n + (size_t)(hbY + g) * w + x0,
                                      Os + (size_t)g * L.ROS + m * L.PB, bytes);
                }
                asm volatile("cp.async.bulk.commit_group;" ::: "memory");
            }
        } else if (hbN > 0 && tid < TW && x0 + tid < w) {
            float* d[NAB];
#pragma unroll
            for (int m = 0; m < NAB; ++m) d[m] = dstimg + (size_t)m * n + (size_t)hbY * w + x0 + tid;
            const float* os = Os + tid;
            for (int g = 0; g < hbN; ++g) {
#pragma unroll
                for (int m = 0; m < NAB; ++m) {
                    *d[m] = os[m * PB];
                    d[m] += w;
                }
                os += L.ROS;
            }
        }
        hbN = 0;
        if (yb >= yB1) break;
        yA += nA;
        sA += nA;
        if (sA >= RBA) sA -= RBA;

        // ================= X: column phases
        // stage B: outputs whose a, b windows [y - R, y + R] are complete (rows < yA)
        const int allowed = (yA >= yA1) ? yB1 : min(yB1, yA - R);
        const int nB = min(G, allowed - yb);
        if (nB > 0) {
            if (colBv) {
                // row y of the a, b ring (y >= yA - RBA): float offset of its slot
                const int rstep = L.RAB, rlen = RBA * L.RAB;
                auto slot_off = [&](int y) {
                    int s = sA - (yA - y);
                    s = s < 0 ? s + RBA : s;
                    return s * rstep;
                };
                const float* abc = ABr + tid;
                if (yb == y0) {                   // warm-up: window of y0 - 1
                    for (int y = max(0, y0 - R - 1); y < min(h, y0 + R); ++y) {
                        const float* r = abc + slot_off(y);
#pragma unroll
                        for (int m = 0; m < NAB; ++m) accB[m] += r[m * PA];
                    }
                }
                int oa = slot_off(min(yb + R, h - 1));
                int os_ = slot_off(max(yb - R - 1, 0));
                float* vcol = VsB + tid;
                const bool full = nB == G && yb - R - 1 >= 0 && yb + G - 1 + R < h;
                if (full) {
                    // interior batch: straight-line code, ring wrap tested once per row
#pragma unroll
                    for (int g = 0; g < G; ++g) {
#pragma unroll
                        for (int m = 0; m < NAB; ++m) accB[m] += abc[oa + m * PA] - abc[os_ + m * PA];
                        float* v = vcol + g * L.RVB;
#pragma unroll
                        for (int m = 0; m < NAB; ++m) {
                            *v = accB[m];
                            v += VPB;
                        }
                        oa += rstep;
                        oa = oa >= rlen ? oa - rlen : oa;
                        os_ += rstep;
                        os_ = os_ >= rlen ? os_ - rlen : os_;
                    }
                }
#pragma unroll
                for (int g = 0; g < G; ++g) {
                    if (!full && g < nB) {
                        const int y = yb + g;
                        const bool hasA = y + R < h, hasS = y - R - 1 >= 0;
#pragma unroll
                        for (int m = 0; m < NAB; ++m)
                            accB[m] += (hasA ? abc[oa + m * PA] : 0.0f) - (hasS ? abc[os_ + m * PA] : 0.0f);
#pragma unroll
                        for (int m = 0; m < NAB; ++m) vcol[g * L.RVB + m * VPB] = accB[m];
                        if (hasA) { oa += rstep; if (oa >= rlen) oa -= rlen; }
                        if (hasS) { os_ += rstep; if (os_ >= rlen) os_ -= rlen; }
                    }
                }
            }
            hbY = yb;
            hbN = nB;
            yb += nB;
        }
        // stage A: the next batch of a, b rows
        nA = max(0, min(G, yA1 - yA));
        if (nA > 0) {
            column_A(yA, nA);
            load_batch(yA + nA);
        }
        // the bulk copies of the previous outputs have read Os before the next Y phase rewrites it
        if (P.bulk_out && tid == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
        __syncthreads();
    }
    if (P.bulk_out && tid == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

}  // namespace fgf
