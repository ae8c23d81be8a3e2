// k4_variants.cuh -- K4 variants kept for the development microbenchmark (tools/k4_bench.cu)
// only: a persistent column walker with double-buffered staging and a TMA bulk-copy pipeline.
// Both measured slower than the cp.async-ring output_async_kernel the library launches
// (profiles/round1/k4_microbench.txt), so they are not part of libfgf.so.
#pragma once
#include "../paper_1505_00996_b200/csrc/fgf_kernels.cuh"

namespace fgf {

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
    using V = Vec<float, PX>;
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
        return static_cast<const float*>(P.I) + (size_t)img * CI * N + (size_t)Yb * W + X;
    };
    auto q_base = [&](int item) {
        const int img = item / bands, Yb = (item % bands) * TR;
        return static_cast<float*>(P.q) + (size_t)img * CP * N + (size_t)Yb * W + X;
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
