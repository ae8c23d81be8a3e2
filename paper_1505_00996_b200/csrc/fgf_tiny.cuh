// fgf_tiny.cuh -- K6: the whole Fast Guided Filter (Alg. 2) for ONE small
// gray image per CTA group, in ONE kernel, for single-image latency (BASELINE.json config 0:
// 256 x 256, r = 8, s = 4 -> a 64 x 64 low-res image).
//
// The low-res image (h w <= 4096 samples) fits in shared memory, so the chain needs no running
// sums and no streaming.  Each CTA owns a band of ~16 full-resolution output rows and computes
// the chain only on the low-res rows its band needs (mean maps on the band's source rows
// [ylo, yhi] of R5, a, b r' rows further, samples 2r' rows further), loading their samples at
// once (one memory round trip):
//   step 1  I', p' (nearest R3, or the clipped s x s block mean R4, fp64 sum as K0)
//   step 2  horizontal then vertical clipped window sums of I', I'^2, p', I'p' in fp64 (R1)
//   steps 3-4  var, cov (fp64), a = cov / (var + eps) (fp32 quotient), b
//   step 5  box of a, b (horizontal, then vertical; fp32 sums of <= 17 fp32 values)
// redundantly (it is a few microseconds of work), then writes its own band of full-resolution
// output rows: the bilinear upsample of mean_a, mean_b (R5, exact integer source coordinates)
// times the full-resolution I plus mean_b (steps 6-7).  Direct window sums cost
// O(r') per sample, so K6 serves r' <= 8 only.
//
// Nothing here is shared with oracle/ (the independent CPU reference).
#pragma once

#include <cuda_runtime.h>

#include "fgf_kernels.cuh"

namespace fgf {

constexpr int kTinyMaxN = 4096;      // low-res samples per image
constexpr int kTinyMaxR = 8;
constexpr int kTinyThreads = 512;

struct TinyParams {
    const float* I;        // [img][H][W]
    const float* p;        // [img][H][W] (may equal I)
    float* q;              // [img][H][W]
    int H, W, h, w, s, sub, R;
    int bands;             // CTAs per image: output rows [b H / bands, (b + 1) H / bands)
    double eps;
    float k1, k0;          // mean maps as written: k1 mean_a + k0, k1 mean_b (enhance fold)
};

// dynamic smem: Is, ps [n] fp32; Hs [4][n] fp64 (window sums, then the box of a, b);
// A, B [n] fp32 (a, b, then mean_a, mean_b).
inline size_t tiny_smem(int n) { return (size_t)n * (2 * 4 + 4 * 8 + 2 * 4); }

// grid (bands, images), block kTinyThreads.
__global__ void __launch_bounds__(kTinyThreads) tiny_gray_kernel(TinyParams P) {
    extern __shared__ __align__(16) unsigned char smem[];
    const int h = P.h, w = P.w, n = h * w, R = P.R, s = P.s, H = P.H, W = P.W;
    float* Is = reinterpret_cast<float*>(smem);
    float* ps = Is + n;
    double* Hs = reinterpret_cast<double*>(ps + n);     // [4][n]
    float* A = reinterpret_cast<float*>(Hs + 4 * (size_t)n);
    float* B = A + n;
    float* HA = reinterpret_cast<float*>(Hs);           // [2][n] box of a, b (reuses Hs)
    const int tid = threadIdx.x, img = blockIdx.y;
    const float* Ig = P.I + (size_t)img * H * W;
    const float* pg = P.p + (size_t)img * H * W;
    const bool self = P.I == P.p;
    // this CTA's output rows and the low-res rows each stage needs (indices are global rows;
    // the arrays are indexed by row - rs0)
    const int Y0 = (int)((long long)blockIdx.x * H / P.bands);
    const int Y1 = (int)((long long)(blockIdx.x + 1) * H / P.bands);
    int ylo, yhi, yd;
    float fd;
    src_coord(Y0, h, H, ylo, yd, fd);
    src_coord(Y1 - 1, h, H, yd, yhi, fd);
    const int rm0 = ylo, rm1 = yhi + 1;                          // mean maps
    const int ra0 = max(0, rm0 - R), ra1 = min(h, rm1 + R);      // a, b
    const int rs0 = max(0, ra0 - R), rs1 = min(h, ra1 + R);      // samples, statistics
    const int nS = (rs1 - rs0) * w;
    auto L = [&](int y, int x) { return (y - rs0) * w + x; };

    // ---- step 1: samples; nearest: 8 loads of the thread in flight together
    if (P.sub == 0) {
        for (int i0 = tid; i0 < nS; i0 += 8 * kTinyThreads) {
            float vi[8], vp[8];
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                const int i = i0 + k * kTinyThreads;
                const int y = rs0 + i / w, x = i % w;
                const size_t o = (size_t)y * s * W + (size_t)x * s;
                vi[k] = i < nS ? __ldg(Ig + o) : 0.0f;
                vp[k] = (i < nS && !self) ? __ldg(pg + o) : 0.0f;
            }
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                const int i = i0 + k * kTinyThreads;
                if (i < nS) {
                    Is[i] = vi[k];
                    ps[i] = vp[k];
                }
            }
        }
    } else {
        for (int i = tid; i < nS; i += kTinyThreads) {
            const int y = rs0 + i / w, x = i % w;
            const int ya = y * s, yb = min(H, ya + s), xa = x * s, xb = min(W, xa + s);
            double ai = 0.0, ap = 0.0;
            for (int yy = ya; yy < yb; ++yy)
                for (int xx = xa; xx < xb; ++xx) {
                    ai += (double)__ldg(Ig + (size_t)yy * W + xx);
                    if (!self) ap += (double)__ldg(pg + (size_t)yy * W + xx);
                }
            const double c = (double)((yb - ya) * (xb - xa));
            Is[i] = (float)(ai / c);
            ps[i] = (float)(ap / c);
        }
    }
    __syncthreads();
    const float* pv = self ? Is : ps;

    // ---- step 2a: horizontal window sums (fp64; products of two floats are exact)
    for (int i = tid; i < nS; i += kTinyThreads) {
        const int yl = i / w, x = i % w;
        double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
        for (int xx = max(0, x - R); xx <= min(w - 1, x + R); ++xx) {
            const double a = (double)Is[yl * w + xx], b = (double)pv[yl * w + xx];
            s0 += a;
            s1 = fma(a, a, s1);
            s2 += b;
            s3 = fma(a, b, s3);
        }
        Hs[i] = s0;
        Hs[n + i] = s1;
        Hs[2 * n + i] = s2;
        Hs[3 * n + i] = s3;
    }
    __syncthreads();
    // ---- step 2b + 3-4: vertical sums, means, coefficients (a, b rows [ra0, ra1))
    for (int i = tid; i < (ra1 - ra0) * w; i += kTinyThreads) {
        const int y = ra0 + i / w, x = i % w;
        const int y0 = max(0, y - R), y1 = min(h - 1, y + R);
        double S0 = 0.0, S1 = 0.0, S2 = 0.0, S3 = 0.0;
        for (int yy = y0; yy <= y1; ++yy) {
            const int j = L(yy, x);
            S0 += Hs[j];
            S1 += Hs[n + j];
            S2 += Hs[2 * n + j];
            S3 += Hs[3 * n + j];
        }
        const int cx = min(w - 1, x + R) - max(0, x - R) + 1;
        const double inv = 1.0 / (double)((y1 - y0 + 1) * cx);
        const double mI = S0 * inv, mp = S2 * inv;
        double var = fma(-mI, mI, S1 * inv);                 // var_I
        var = var < 0.0 ? 0.0 : var;                         // R8
        const double cov = fma(-mI, mp, S3 * inv);           // cov_Ip
        const float a = (float)cov / (float)(var + P.eps);   // Eq.2
        A[L(y, x)] = a;
        B[L(y, x)] = fmaf(-a, (float)mI, (float)mp);         // Eq.3
    }
    __syncthreads();
    // ---- step 5a: horizontal box of a, b
    for (int i = tid; i < (ra1 - ra0) * w; i += kTinyThreads) {
        const int y = ra0 + i / w, x = i % w;
        float sa = 0.0f, sb = 0.0f;
        for (int xx = max(0, x - R); xx <= min(w - 1, x + R); ++xx) {
            sa += A[L(y, xx)];
            sb += B[L(y, xx)];
        }
        HA[L(y, x)] = sa;
        HA[n + L(y, x)] = sb;
    }
    __syncthreads();
    // ---- step 5b: vertical box -> mean_a, mean_b on rows [rm0, rm1) (into A, B; the
    // enhance fold applied)
    for (int i = tid; i < (rm1 - rm0) * w; i += kTinyThreads) {
        const int y = rm0 + i / w, x = i % w;
        const int y0 = max(0, y - R), y1 = min(h - 1, y + R);
        float sa = 0.0f, sb = 0.0f;
        for (int yy = y0; yy <= y1; ++yy) {
            sa += HA[L(yy, x)];
            sb += HA[n + L(yy, x)];
        }
        const int cx = min(w - 1, x + R) - max(0, x - R) + 1;
        const float inv = 1.0f / (float)((y1 - y0 + 1) * cx);
        A[L(y, x)] = fmaf(P.k1, sa * inv, P.k0);
        B[L(y, x)] = P.k1 * (sb * inv);
    }
    __syncthreads();
    // ---- steps 6-7: this CTA's band of output rows, 8 rows per group: the 8 guidance loads of a
    // thread in flight together, then the outputs
    float* qg = P.q + (size_t)img * H * W;
    for (int Yg = Y0; Yg < Y1; Yg += 8) {
        for (int X = tid; X < W; X += kTinyThreads) {
            int xa, xb;
            float fx;
            src_coord(X, w, W, xa, xb, fx);
            float Iv[8];
#pragma unroll
            for (int k = 0; k < 8; ++k) Iv[k] = Yg + k < Y1 ? __ldg(Ig + (size_t)(Yg + k) * W + X) : 0.0f;
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                const int Y = Yg + k;
                if (Y < Y1) {
                    int ya, yb;
                    float fy;
                    src_coord(Y, h, H, ya, yb, fy);
                    const int la = L(ya, 0), lb = L(yb, 0);
                    auto bil = [&](const float* M) {
                        const float t0 = fmaf(fx, M[la + xb] - M[la + xa], M[la + xa]);
                        const float t1 = fmaf(fx, M[lb + xb] - M[lb + xa], M[lb + xa]);
                        return fmaf(fy, t1 - t0, t0);
                    };
                    __stcs(qg + (size_t)Y * W + X, fmaf(bil(A), Iv[k], bil(B)));
                }
            }
        }
    }
}

}  // namespace fgf
