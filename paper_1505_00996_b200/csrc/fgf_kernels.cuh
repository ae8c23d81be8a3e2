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

#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace fgf {

enum { MODE_STATS = 0, MODE_MEAN = 1 };

// Packed PX-element vectors of the I / q element type E (float, __half, __nv_bfloat16,
// unsigned char) as raw
// 32-bit words: one streaming load / store per thread and row, elements converted to fp32
// (reduced-precision I/O: storage only, every operation is fp32).
template <int BYTES> struct RawT;
template <> struct RawT<16> { using T = uint4; };
template <> struct RawT<8> { using T = uint2; };
template <> struct RawT<4> { using T = unsigned int; };
template <> struct RawT<2> { using T = unsigned short; };
template <> struct RawT<1> { using T = unsigned char; };
__device__ __forceinline__ unsigned raw_word(const uint4& r, int k) {
    return k == 0 ? r.x : (k == 1 ? r.y : (k == 2 ? r.z : r.w));
}
__device__ __forceinline__ unsigned raw_word(const uint2& r, int k) { return k == 0 ? r.x : r.y; }
__device__ __forceinline__ unsigned raw_word(unsigned r, int) { return r; }
__device__ __forceinline__ unsigned raw_word(unsigned short r, int) { return r; }
__device__ __forceinline__ unsigned raw_word(unsigned char r, int) { return r; }
__device__ __forceinline__ void raw_make(uint4& r, const unsigned* w) { r = make_uint4(w[0], w[1], w[2], w[3]); }
__device__ __forceinline__ void raw_make(uint2& r, const unsigned* w) { r = make_uint2(w[0], w[1]); }
__device__ __forceinline__ void raw_make(unsigned& r, const unsigned* w) { r = w[0]; }
__device__ __forceinline__ void raw_make(unsigned short& r, const unsigned* w) { r = (unsigned short)w[0]; }
__device__ __forceinline__ void raw_make(unsigned char& r, const unsigned* w) { r = (unsigned char)w[0]; }

template <typename E> struct ElemT;
template <> struct ElemT<float> {
    __device__ static float f(unsigned b) { return __uint_as_float(b); }
    __device__ static unsigned bits(float x) { return __float_as_uint(x); }
    __device__ static float load(const float* p) { return __ldg(p); }
};
template <> struct ElemT<__half> {
    __device__ static float f(unsigned b) { return __half2float(__ushort_as_half((unsigned short)b)); }
    __device__ static unsigned bits(float x) { return __half_as_ushort(__float2half_rn(x)); }
    __device__ static float load(const __half* p) { return __half2float(__ldg(p)); }
};
template <> struct ElemT<__nv_bfloat16> {
    __device__ static float f(unsigned b) { return __uint_as_float(b << 16); }
    __device__ static unsigned bits(float x) { return __bfloat16_as_ushort(__float2bfloat16_rn(x)); }
    __device__ static float load(const __nv_bfloat16* p) { return __bfloat162float(__ldg(p)); }
};
// 8-bit codes (R19): code k is the value fl(k x fl(1/255)) (one fp32 product, within
// an ulp of k / 255); a value is stored as the code nearest to 255 x, saturated to [0, 255].
template <> struct ElemT<unsigned char> {
    __device__ static float f(unsigned b) { return __fmul_rn((float)(b & 0xffu), 1.0f / 255.0f); }
    __device__ static unsigned bits(float x) {
        return __float2uint_rn(fminf(fmaxf(x * 255.0f, 0.0f), 255.0f));
    }
    __device__ static float load(const unsigned char* p) { return f(__ldg(p)); }
};

template <typename E, int PX>
struct Vec {
    static constexpr int EB = (int)sizeof(E), BYTES = PX * EB;
    using T = typename RawT<BYTES>::T;
    __device__ static T ld(const E* p) { return __ldcs(reinterpret_cast<const T*>(p)); }
    __device__ static float get(const T& v, int i) {
        const int bit = i * EB * 8;
        const unsigned w = raw_word(v, bit >> 5) >> (bit & 31);
        return ElemT<E>::f(EB == 4 ? w : (w & ((1u << (EB * 8)) - 1u)));
    }
    __device__ static void st(E* p, const float* v) {
        unsigned w[BYTES >= 4 ? BYTES / 4 : 1] = {};
#pragma unroll
        for (int i = 0; i < PX; ++i) {
            const int bit = i * EB * 8;
            w[bit >> 5] |= ElemT<E>::bits(v[i]) << (bit & 31);
        }
        T r;
        raw_make(r, w);
        __stcs(reinterpret_cast<T*>(p), r);
    }
};



// ------------------------------------------------------------------ K0: block-mean subsample

struct SubParams {
    const void* src;        // [plane][H][W] of the I/O element type E
    float* dst;             // [plane][h][w]
    int H, W, h, w, s;
    int rows_per_cta;       // low-res rows per CTA (grid-y covers h / rows_per_cta)
    const void* src2;       // planes >= nsplit come from src2 (one launch for I and p)
    int nsplit;
};

// Source plane `plane` of a K0 launch (two inputs in one grid: src, then src2).
template <typename E>
__device__ __forceinline__ const E* sub_src(const SubParams& P, size_t plane) {
    const size_t HW = (size_t)P.H * P.W;
    return plane < (size_t)P.nsplit ? static_cast<const E*>(P.src) + plane * HW
                                    : static_cast<const E*>(P.src2) + (plane - P.nsplit) * HW;
}

// R4: mean of the clipped s x s block, summed in fp64.  One thread per
// low-res column, several low-res rows per CTA for memory-level parallelism.
// grid (ceil(w/256), ceil(h/rows_per_cta), planes).
template <bool VEC4, typename E = float>
__global__ void __launch_bounds__(256) subsample_block_kernel(SubParams P) {
    const int x = blockIdx.x * blockDim.x + threadIdx.x;
    if (x >= P.w) return;
    const size_t plane = blockIdx.z;
    const E* src = sub_src<E>(P, plane);
    float* dst = P.dst + plane * (size_t)P.h * P.w;
    const int y0 = blockIdx.y * P.rows_per_cta;
    const int y1 = min(P.h, y0 + P.rows_per_cta);
    const int xa = x * P.s, xb = min(P.W, xa + P.s);
    for (int y = y0; y < y1; ++y) {
        const int ya = y * P.s, yb = min(P.H, ya + P.s);
        double acc = 0.0;
        if (VEC4) {  // s == 4, W % 4 == 0, rows aligned to 4 elements
            using V = Vec<E, 4>;
            for (int yy = ya; yy < yb; ++yy) {
                const typename V::T v = V::ld(src + (size_t)yy * P.W + 4 * x);
#pragma unroll
                for (int i = 0; i < 4; ++i) acc += (double)V::get(v, i);
            }
        } else {
            for (int yy = ya; yy < yb; ++yy) {
                const E* row = src + (size_t)yy * P.W;
                for (int xx = xa; xx < xb; ++xx) acc += (double)ElemT<E>::load(row + xx);
            }
        }
        dst[(size_t)y * P.w + x] = (float)(acc / (double)((yb - ya) * (xb - xa)));
    }
}

// R3: nearest = top-left sample I[y*s][x*s], compacted into low-res planes so
// that the box engine's repeated row reads (warm-up, subtracted rows) touch 4 bytes per
// sample instead of a 32-byte sector.  RPC rows per thread, loads issued before stores.
// grid (ceil(w/256), ceil(h/RPC), planes).
template <int RPC, typename E = float>
__global__ void __launch_bounds__(256) subsample_nearest_kernel(SubParams P) {
    const int x = blockIdx.x * blockDim.x + threadIdx.x;
    if (x >= P.w) return;
    const size_t plane = blockIdx.z;
    const E* src = sub_src<E>(P, plane) + (size_t)x * P.s;
    float* dst = P.dst + plane * (size_t)P.h * P.w + x;
    const int y0 = blockIdx.y * RPC;
    float v[RPC];
#pragma unroll
    for (int k = 0; k < RPC; ++k)
        if (y0 + k < P.h) v[k] = ElemT<E>::load(src + (size_t)(y0 + k) * P.s * P.W);
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
    // MEAN only: groups > 1 splits the maps of each image into `groups` launches-in-one of
    // NIN consecutive planes (blockIdx.z = image * groups + group; group g reads planes and
    // writes maps [g NIN, (g + 1) NIN) and folds k0 into its map g).
    int groups;
};

// Rows per batch G (each warp slides along one row of a batch), odd run length K, smem.
// G_ / MINB_ override the defaults (development microbenchmark).
template <int MODE, int CI, int CP, int NT, int G_ = 0, int MINB_ = 0>
struct StripConfig {
    using T = StripTraits<MODE, CI, CP>;
    static constexpr int NMAP = T::NMAP;
    static constexpr int NOUT = T::NOUT;
    static constexpr int NW = NT / 32;
    static constexpr int VPMAX = NT == 64 ? 128 : (NT == 128 ? 256 : (NT == 256 ? 448 : 992));   // worst-case padded row
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
                                int ostride, int grp) {
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
                                int ostride, int grp) {
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
                                int ostride, int grp) {
#pragma unroll
        for (int m = 0; m < (CI + 1) * CP; ++m) {
            const int c = m / (CI + 1), j = m - c * (CI + 1);
            // grouped launch (one p channel per CTA, CP = 1 here): channel grp's diagonal
            dst[m * ostride] = fmaf(P.k1, (float)(S[m] * inv), j == c + grp ? P.k0 : 0.0f);
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
// HPRE: wide windows (large r') -- the horizontal window sums come from an in-place prefix
// sum of each snapshotted row (one warp per row; cost independent of r') instead of sliding
// runs whose restart costs 2r'+1 reads per run.  Sums of fp64 column sums over <= 1024
// columns: the difference of two prefixes loses nothing at the 1e-4 level.
template <int MODE, int CI, int CP, int NT, int G_ = 0, int MINB_ = 0, bool HPRE = false>
__global__ void __launch_bounds__(NT, (StripConfig<MODE, CI, CP, NT, G_, MINB_>::MINB)) box_strip_kernel(StripParams P) {
    using T = StripTraits<MODE, CI, CP>;
    using C = StripConfig<MODE, CI, CP, NT, G_, MINB_>;
    constexpr int NMAP = T::NMAP;
    constexpr int NIN = T::NIN;
    constexpr int NOUT = T::NOUT;
    constexpr int G = C::G;
    constexpr int K = C::K;
    extern __shared__ double smem_d[];
    // box of a, b: a programmatic dependent (K4, run_all) may start its map-independent
    // prologue once every CTA of this grid is running (no-op otherwise)
    if (MODE == MODE_MEAN) asm volatile("griddepcontrol.launch_dependents;");
    const int VP = P.VP;
    double* Vs = smem_d;                                                  // [G][NMAP][VP]
    float* Os = reinterpret_cast<float*>(Vs + (size_t)G * NMAP * VP);      // [G][NOUT][NT]
    double* invx = reinterpret_cast<double*>(Os + (size_t)G * NOUT * NT);  // [NT]

    const int tid = threadIdx.x;
    const int groups = P.groups > 1 ? P.groups : 1;
    const int img = blockIdx.z / groups, grp = blockIdx.z - img * groups;
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
    const float* bI = P.srcI + img * P.imgI + (long long)grp * NIN * planeI;
    const float* bP = (MODE == MODE_STATS) ? P.srcP + img * P.imgP : bI;
    float* dst = P.dst + ((size_t)img * groups + grp) * NOUT * n + x0;

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

        if (HPRE) {
            // ---- horizontal phase by prefix sums: rows (g, m), one warp each, in place over
            // Vs indices [0, L); the window of output oc is P[cbase+oc+2R] - P[cbase+oc-1].
            const int L = R + ncol;
            const int CH = (L + 31) >> 5;
            const int nrows_b = min(G, ye - yb);
            for (int rr = warp; rr < nrows_b * NMAP; rr += C::NW) {
                double* vrow = Vs + (size_t)rr * VP;
                const int a = lane * CH, e = min(L, a + CH);
                double tot = 0.0;
                for (int i = a; i < e; ++i) tot += vrow[i];
                // exclusive warp scan of the chunk totals
                double x = tot;
#pragma unroll
                for (int d = 1; d < 32; d <<= 1) {
                    const double y = __shfl_up_sync(0xffffffffu, x, d);
                    if (lane >= d) x += y;
                }
                double run = x - tot;
                for (int i = a; i < e; ++i) {
                    run += vrow[i];
                    vrow[i] = run;
                }
            }
            __syncthreads();
            for (int qq = tid; qq < nrows_b * ocn; qq += NT) {
                const int g = qq / ocn, oc = qq - g * ocn;
                const int yo2 = yb + g;
                const double invy = 1.0 / (double)(min(h - 1, yo2 + R) - max(0, yo2 - R) + 1);
                // past the scanned range the columns are zero pads: the prefix stays P[L-1]
                const int hi = min(cbase + oc + 2 * R, L - 1), lo = cbase + oc - 1;
                const double* pr = Vs + (size_t)g * NMAP * VP;
                double S[NMAP];
#pragma unroll
                for (int m = 0; m < NMAP; ++m)
                    S[m] = pr[m * VP + hi] - (lo >= 0 ? pr[m * VP + lo] : 0.0);
                StripEpilogue<MODE, CI, CP>::emit(S, invx[oc] * invy, P,
                                                  Os + (size_t)g * NOUT * NT + oc, NT, grp);
            }
        }
        // ---- horizontal phase: branch-free sliding window along each snapshotted row.
        const int yo = yb + hg;
        if (!HPRE && yo < ye && oc0 < ocn) {
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
                    StripEpilogue<MODE, CI, CP>::emit(S, invx[oc0 + i] * invy, P, orow + i, NT, grp);
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

// cp.async helpers (K4 staging and rings)
__device__ __forceinline__ void cp_async4(float* dst, const float* src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"((uint32_t)__cvta_generic_to_shared(dst)),
                 "l"(src)
                 : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }

template <int BYTES>
__device__ __forceinline__ void cp_async_px(void* dst, const void* src) {
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


// Stage the low-res rectangle rows [ylo, ylo + nrl) x columns [x4, x4 + ncs) of the NC maps
// into Ms[(row * NC + map) * ncs + col] with cp.async (all copies in flight at once, no
// register round trip; the caller commits and waits).  x4 is 4-aligned and ncs a multiple of
// 4: with w % 4 == 0 and a 16-byte aligned maps pointer every line moves in 16-byte copies,
// otherwise in 4-byte copies clipped at the image edge.  One warp per line.
template <int NC, int NT>
__device__ __forceinline__ void stage_rect(float* Ms, const float* Mb, size_t n, int w, int ylo,
                                           int nrl, int x4, int ncs, int tid) {
    const int lane = tid & 31;
    if ((w & 3) == 0 && (reinterpret_cast<uintptr_t>(Mb) & 15u) == 0) {
        const int nq = ncs >> 2;
        for (int rm = tid >> 5; rm < nrl * NC; rm += NT / 32) {
            const int rr = rm / NC, m = rm - rr * NC;
            const float* src = Mb + (size_t)m * n + (size_t)(ylo + rr) * w + x4;
            float* d = Ms + (size_t)rm * ncs;
            for (int c = lane; c < nq; c += 32) cp_async_px<16>(d + 4 * c, src + 4 * c);
        }
    } else {
        const int cols = min(ncs, w - x4);
        for (int rm = tid >> 5; rm < nrl * NC; rm += NT / 32) {
            const int rr = rm / NC, m = rm - rr * NC;
            const float* src = Mb + (size_t)m * n + (size_t)(ylo + rr) * w + x4;
            float* d = Ms + (size_t)rm * ncs;
            for (int c = lane; c < cols; c += 32) cp_async_px<4>(d + c, src + c);
        }
    }
}

// ------------------------------------------------------------------ K4: upsample + output

struct OutParams {
    const void* I;         // [img][CI][H][W] of the I/O element type E   (H rows of the image, or of a row band)
    const float* M;        // [img][(CI+1)CP][hm][w] mean maps (hm low-res rows)
    void* q;               // [img][CP][H][W] of E
    int H, W, hm, w;       // local buffer geometry
    int Hg, hg;            // global full-res / low-res heights (the vertical map, R5)
    int Yoff, yoff;        // global row of local row 0 of I/q, and of the maps buffer
    int TR;                // full-resolution rows walked by each thread
    int pdl;               // 1: launched as a programmatic dependent of the kernel writing M --
                           // the guidance rows are prefetched before griddepcontrol.wait, the
                           // maps staged after it (output_async_kernel)
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
template <int CI, int CP, int PX, bool S1, int U_ = 0, int MINB_ = 0, int ABL = 0,
          typename E = float>
__global__ void __launch_bounds__(256, (MINB_ ? MINB_ : OutCfg<CI, CP, PX>::MINB)) output_kernel(OutParams P) {
    constexpr int NC = OutCfg<CI, CP, PX>::NC;
    constexpr int U = U_ ? U_ : OutCfg<CI, CP, PX>::U;
    constexpr int NM = S1 ? NC : 1;              // map planes streamed per row (S1)
    using V = Vec<E, PX>;                        // I, q
    using VT = typename V::T;
    using VM = Vec<float, PX>;                   // maps (S1)
    using VMT = typename VM::T;
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
    const E* Ip = static_cast<const E*>(P.I) + (size_t)img * CI * N + (size_t)Y0 * W + X;
    E* qp = static_cast<E*>(P.q) + (size_t)img * CP * N + (size_t)Y0 * W + X;
    const float* Mb = P.M + (size_t)img * NC * n;
    // S1 only: the maps have the image's geometry, shifted by the band offsets
    const float* Mp = Mb + (size_t)(P.Yoff + Y0 - P.yoff) * W + X;

    // Issue the first U rows before anything else: I planes, and (S1) the coefficient maps.
    VT cur[U][CI];
    VMT curm[U][NM];
#pragma unroll
    for (int u = 0; u < U; ++u)
        if (act && u < nrows) {
#pragma unroll
            for (int j = 0; j < CI; ++j) cur[u][j] = V::ld(Ip + (size_t)u * W + (size_t)j * N);
            if (S1)
#pragma unroll
                for (int m = 0; m < NM; ++m) curm[u][m] = VM::ld(Mp + (size_t)u * W + (size_t)m * n);
        }

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
        xlo &= ~3;
        ncl = (xhi + 1 - xlo + 3) & ~3;   // row stride of the staged rectangle
        stage_rect<NC, 256>(Ms, Mb, n, w, ylo, nrl, xlo, ncl, threadIdx.x);
        cp_async_commit();
#pragma unroll
        for (int i = 0; i < PX; ++i) {
            src_coord(min(X + i, W - 1), w, W, oa[i], ob[i], fx[i]);
            oa[i] -= xlo;      // local columns in the staged rectangle
            ob[i] -= xlo;
        }
        cp_async_wait<0>();
        __syncthreads();
    }

    const E* Ipf = Ip + (size_t)U * W;
    const float* Mpf = Mp + (size_t)U * W;
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
                            acc = VM::get(curm[u][S1 ? mb + CI : 0], i);
#pragma unroll
                            for (int j = 0; j < CI; ++j)
                                acc = fmaf(VM::get(curm[u][S1 ? mb + j : 0], i), V::get(cur[u][j], i), acc);
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
                if (t + U < nrows) {
#pragma unroll
                    for (int j = 0; j < CI; ++j) cur[u][j] = V::ld(Ipf + (size_t)j * N);
                    if (S1)
#pragma unroll
                        for (int m = 0; m < NM; ++m) curm[u][m] = VM::ld(Mpf + (size_t)m * n);
                }
                Ipf += W;
                Mpf += W;
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

template <int CI, int CP, int PX, typename E = float>
struct AsyncCfg {
    static constexpr int NC = (CI + 1) * CP;
    static constexpr int U = 8;                                  // rows in flight (power of 2)
    static constexpr int MINB = NC * PX <= 8 ? 4 : 2;
    static constexpr size_t RING_BYTES = (size_t)U * CI * 256 * PX * sizeof(E);
};

// E: element type of I and q (float, __half, __nv_bfloat16); PX * sizeof(E) in {4, 8, 16}.
template <int CI, int CP, int PX, typename E = float>
__global__ void __launch_bounds__(256, (AsyncCfg<CI, CP, PX, E>::MINB)) output_async_kernel(OutParams P) {
    using C = AsyncCfg<CI, CP, PX, E>;
    constexpr int NC = C::NC;
    constexpr int U = C::U;
    using V = Vec<E, PX>;
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
    const E* Ip = static_cast<const E*>(P.I) + (size_t)img * CI * N + (size_t)Y0 * W + X;
    E* qp = static_cast<E*>(P.q) + (size_t)img * CP * N + (size_t)Y0 * W + X;
    const float* Mb = P.M + (size_t)img * NC * n;

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
    xlo &= ~3;
    const int nrl = yhi - ylo + 1, ncl = (xhi + 1 - xlo + 3) & ~3;
    // Issue the first U rows (one commit group per row, empty groups keep the count uniform).
    auto issue_rows = [&] {
#pragma unroll
        for (int u = 0; u < U; ++u) {
            if (act && u < nrows)
#pragma unroll
                for (int j = 0; j < CI; ++j)
                    cp_async_px<V::BYTES>(&ring[(u * CI + j) * 256 + tid], Ip + j * N + (size_t)u * W);
            cp_async_commit();
        }
    };
    if (P.pdl) {
        // programmatic dependent of the low-res chain: everything that does not read the
        // maps (row table, coordinates, the first U guidance rows) overlaps its tail; the
        // maps are staged once it has completed
        issue_rows();
        asm volatile("griddepcontrol.wait;" ::: "memory");
        stage_rect<NC, 256>(Ms, Mb, n, w, ylo, nrl, xlo, ncl, tid);
        cp_async_commit();
    } else {
        stage_rect<NC, 256>(Ms, Mb, n, w, ylo, nrl, xlo, ncl, tid);   // commit group 0
        cp_async_commit();
        issue_rows();
    }
    int oa[PX], ob[PX];
    float fx[PX];
#pragma unroll
    for (int i = 0; i < PX; ++i) {
        src_coord(min(X + i, W - 1), w, W, oa[i], ob[i], fx[i]);
        oa[i] -= xlo;
        ob[i] -= xlo;
    }
    // the rectangle has landed: group 0, or (pdl) the last group
    if (P.pdl) cp_async_wait<0>();
    else cp_async_wait<U>();
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
    const E* Ipf = Ip + (size_t)U * W;
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
                    cp_async_px<V::BYTES>(&ring[(slot * CI + j) * 256 + tid], Ipf + j * N);
        }
        cp_async_commit();
        qp += W;
        Ipf += W;
    }
    cp_async_wait<0>();
}

// ------------------------------------------------------------------ K4, channel split
//
// Colour guidance with several p channels (NC = 4 C_p maps).  One thread per (output channel
// c, 4-pixel group) keeps the interpolated rows of only its channel's C_I + 1 maps and
// writes q_c, instead of one thread per pixel carrying all NC maps.  The guidance rows stream
// through ONE shared ring per CTA, each float4 loaded once by cp.async (64 * C_I loads per
// row spread over the CTA); completion is tracked per slot by an mbarrier that every thread
// arrives on when its copies land ("full"), and slot reuse by a second mbarrier every thread
// arrives on after reading the row ("empty"); a slot is refilled one row late so the empty
// wait rarely blocks.  CTA: 64 groups x C_p channels, 256 pixels wide.
template <int CI, int CP>
struct SplitCfg {
    static constexpr int NC = (CI + 1) * CP;
    static constexpr int PX = 4;
    static constexpr int NT = 64 * CP;
    static constexpr int U = 8;
    static constexpr size_t RING_BYTES = (size_t)U * CI * 64 * PX * 4;   // + 2U mbarriers
    static constexpr size_t BAR_BYTES = 2 * U * 8;
};

__device__ __forceinline__ uint32_t smem_addr(const void* p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init_cta(uint64_t* bar, int count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_arrive_cta(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_addr(bar)) : "memory");
}
// arrive once this thread's earlier cp.async copies have landed (count not incremented)
__device__ __forceinline__ void cp_async_mbar_arrive(uint64_t* bar) {
    asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_addr(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait_parity(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "WAITP_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAITP_%=;\n}" ::"r"(smem_addr(bar)),
        "r"(parity)
        : "memory");
}

template <int CI, int CP>
__global__ void __launch_bounds__(SplitCfg<CI, CP>::NT) output_split_kernel(OutParams P) {
    using C = SplitCfg<CI, CP>;
    constexpr int NC = C::NC, PX = C::PX, NT = C::NT, U = C::U, NM = CI + 1;
    constexpr int LOADS = 64 * CI;                                // float4 per ring row
    using V = Vec<float, PX>;
    using VT = typename V::T;
    __shared__ int s_ya[kMaxTR];
    __shared__ int s_y1[kMaxTR];
    __shared__ float s_fy[kMaxTR];
    extern __shared__ __align__(16) float smx[];
    uint64_t* full = reinterpret_cast<uint64_t*>(smx);            // [U]
    uint64_t* empty = full + U;                                   // [U]
    VT* ring = reinterpret_cast<VT*>(smx + C::BAR_BYTES / 4);     // [U][CI][64]
    float* Ms = smx + (C::BAR_BYTES + C::RING_BYTES) / 4;         // [nrl][NC][ncl]
    const int H = P.H, W = P.W, h = P.hm, w = P.w;
    const int tid = threadIdx.x;
    const int ch = tid >> 6, g = tid & 63;                        // output channel, pixel group
    const int Y0 = blockIdx.y * P.TR;
    const int nrows = min(P.TR, H - Y0);
    const int X0 = blockIdx.x * 64 * PX;
    const bool act = X0 + g * PX < W;
    const int X = act ? X0 + g * PX : X0;
    const int img = blockIdx.z;
    const size_t N = (size_t)H * W, n = (size_t)h * w;
    const float* Ib = static_cast<const float*>(P.I) + (size_t)img * CI * N + (size_t)Y0 * W + X0;
    float* qp = static_cast<float*>(P.q) + ((size_t)img * CP + ch) * N + (size_t)Y0 * W + X;
    const float* Mb = P.M + (size_t)img * NC * n;

    if (tid == 0) {
        for (int u = 0; u < U; ++u) {
            mbar_init_cta(&full[u], NT);
            mbar_init_cta(&empty[u], NT);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    // this thread's copies of ring row t: float4 k = tid, tid + NT, ... of [CI][64]
    auto issue = [&](int t) {
        if (t < nrows) {
            const float* rowp = Ib + (size_t)t * W;
            VT* slot = ring + (size_t)(t & (U - 1)) * LOADS;
            for (int k = tid; k < LOADS; k += NT) {
                const int j = k >> 6, gg = k & 63;
                if (X0 + gg * PX < W) cp_async_px<16>(&slot[k], rowp + (size_t)j * N + gg * PX);
            }
        }
        cp_async_mbar_arrive(&full[t & (U - 1)]);
    };

    for (int t = tid; t < nrows; t += NT) {
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
    src_coord(min(W, X0 + 64 * PX) - 1, w, W, xd, xhi, fd);
    xlo &= ~3;
    const int nrl = yhi - ylo + 1, ncl = (xhi + 1 - xlo + 3) & ~3;
    stage_rect<NC, NT>(Ms, Mb, n, w, ylo, nrl, xlo, ncl, tid);
    cp_async_commit();                              // the rectangle: the only commit group
#pragma unroll 1
    for (int u = 0; u < U; ++u) issue(u);           // ring rows: tracked by the full mbarriers
    cp_async_wait<0>();
    int oa[PX], ob[PX];
    float fx[PX];
#pragma unroll
    for (int i = 0; i < PX; ++i) {
        src_coord(min(X + i, W - 1), w, W, oa[i], ob[i], fx[i]);
        oa[i] -= xlo;
        ob[i] -= xlo;
    }
    __syncthreads();

    const int mb = ch * NM;                                       // this channel's maps
    int cy = -2, cy1 = -2;
    float H0[NM][PX], H1[NM][PX], D[NM][PX];
    auto hrow = [&](int y, float (&out)[NM][PX]) {
        const float* mr = Ms + ((size_t)(y - ylo) * NC + mb) * ncl;
#pragma unroll
        for (int m = 0; m < NM; ++m)
#pragma unroll
            for (int i = 0; i < PX; ++i) {
                const float va = mr[m * ncl + oa[i]], vb = mr[m * ncl + ob[i]];
                out[m][i] = fmaf(fx[i], vb - va, va);
            }
    };
    for (int t = 0; t < nrows; ++t) {
        const int ya = s_ya[t];
        const float fy = s_fy[t];
        if (__any_sync(0xffffffffu, ya != cy)) {   // CTA-uniform branch
            if (ya == cy1) {
#pragma unroll
                for (int m = 0; m < NM; ++m)
#pragma unroll
                    for (int i = 0; i < PX; ++i) H0[m][i] = H1[m][i];
            } else {
                hrow(ya, H0);
            }
            cy1 = s_y1[t];
            hrow(cy1, H1);
#pragma unroll
            for (int m = 0; m < NM; ++m)
#pragma unroll
                for (int i = 0; i < PX; ++i) D[m][i] = H1[m][i] - H0[m][i];
            cy = ya;
        }
        const int slot = t & (U - 1);
        mbar_wait_parity(&full[slot], (uint32_t)((t / U) & 1));   // row t landed (all copies)
        if (act) {
            const VT* sr = ring + (size_t)slot * LOADS + g;
            VT iv[CI];
#pragma unroll
            for (int j = 0; j < CI; ++j) iv[j] = sr[j * 64];
            float o[PX];
#pragma unroll
            for (int i = 0; i < PX; ++i) {
                float acc = fmaf(fy, D[CI][i], H0[CI][i]);
#pragma unroll
                for (int j = 0; j < CI; ++j)
                    acc = fmaf(fmaf(fy, D[j][i], H0[j][i]), V::get(iv[j], i), acc);
                o[i] = acc;
            }
            V::st(qp, o);
        }
        mbar_arrive_cta(&empty[slot]);
        // refill the slot read one row ago (everyone is past it by now, so rarely a wait)
        if (t >= 1 && t - 1 + U < nrows) {
            const int s1 = (t - 1) & (U - 1);
            mbar_wait_parity(&empty[s1], (uint32_t)(((t - 1) / U) & 1));
            issue(t - 1 + U);
        }
        qp += W;
    }
    cp_async_wait<0>();
}

}  // namespace fgf
