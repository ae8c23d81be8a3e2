// Microbenchmark of the output pass (K4) variants against plain streaming copies, on
// config-4-shaped data (B x 4096^2 gray, s = 4).  Development tool, not product code.
#include <cstdio>
#include <cstdlib>
#include <vector>
#include "k4_variants.cuh"
using namespace fgf;

template <int UNROLL, bool CS>
__global__ void __launch_bounds__(256) copy_kernel(const float4* __restrict__ a, float4* __restrict__ b, size_t n4) {
    size_t i = (size_t)blockIdx.x * 256 * UNROLL + threadIdx.x;
    const size_t stride = (size_t)gridDim.x * 256 * UNROLL;
    for (; i < n4; i += stride) {
        float4 v[UNROLL];
#pragma unroll
        for (int u = 0; u < UNROLL; ++u)
            if (i + u * 256 < n4) v[u] = CS ? __ldcs(a + i + u * 256) : a[i + u * 256];
#pragma unroll
        for (int u = 0; u < UNROLL; ++u)
            if (i + u * 256 < n4) { if (CS) __stcs(b + i + u * 256, v[u]); else b[i + u * 256] = v[u]; }
    }
}

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); exit(1); } } while (0)

template <typename F>
float timeit(F f, int reps = 5) {
    cudaEvent_t a, b;
    cudaEventCreate(&a); cudaEventCreate(&b);
    f(); CK(cudaDeviceSynchronize());
    cudaEventRecord(a);
    for (int r = 0; r < reps; ++r) f();
    cudaEventRecord(b);
    CK(cudaEventSynchronize(b));
    float ms; cudaEventElapsedTime(&ms, a, b);
    return ms / reps;
}

int main(int argc, char** argv) {
    const int B = argc > 1 ? atoi(argv[1]) : 16;
    const int H = 4096, W = 4096, s = 4, h = H / s, w = W / s;
    const size_t N = (size_t)H * W, n = (size_t)h * w;
    float *I, *q, *M;
    CK(cudaMalloc(&I, B * N * 4)); CK(cudaMalloc(&q, B * N * 4)); CK(cudaMalloc(&M, B * 2 * n * 4));
    CK(cudaMemset(I, 0, B * N * 4)); CK(cudaMemset(M, 0, B * 2 * n * 4));
    int sms = 0; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const double bytes_copy = 2.0 * B * N * 4;
    const double bytes_k4 = 2.0 * B * N * 4 + B * 2 * n * 4;
    const size_t n4 = B * N / 4;
    auto rep = [&](const char* name, float ms, double bytes) {
        printf("%-44s %8.3f ms  %7.1f GB/s  %6.2f us/img\n", name, ms, bytes / ms / 1e6, 1e3 * ms / B);
    };
    for (int g : {sms * 16}) {
        char nm[64];
        snprintf(nm, 64, "copy unroll4 cs grid=%d", g);
        rep(nm, timeit([&] { copy_kernel<4, true><<<g, 256>>>((const float4*)I, (float4*)q, n4); }), bytes_copy);
        snprintf(nm, 64, "copy unroll8 cs grid=%d", g);
        rep(nm, timeit([&] { copy_kernel<8, true><<<g, 256>>>((const float4*)I, (float4*)q, n4); }), bytes_copy);
        snprintf(nm, 64, "copy unroll4 plain grid=%d", g);
        rep(nm, timeit([&] { copy_kernel<4, false><<<g, 256>>>((const float4*)I, (float4*)q, n4); }), bytes_copy);
    }
    rep("cudaMemcpy D2D", timeit([&] { cudaMemcpyAsync(q, I, B * N * 4, cudaMemcpyDeviceToDevice); }), bytes_copy);
    for (int TR : {16, 32, 64}) {
        OutParams op{I, M, q, H, W, h, w, H, h, 0, 0, TR};
        dim3 g4((W + 1023) / 1024, (H + TR - 1) / TR, B);
        const size_t sm = (size_t)(TR / 4 + 3) * 2 * 259 * 4;
        char nm[64];
#define VAR(U, MB) \
        cudaFuncSetAttribute(output_kernel<1, 1, 4, false, U, MB>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100000); \
        snprintf(nm, 64, "walker-staged PX4 U%d MINB%d TR=%d", U, MB, TR); \
        rep(nm, timeit([&] { output_kernel<1, 1, 4, false, U, MB><<<g4, 256, sm>>>(op); }), bytes_k4);
        VAR(2, 4) VAR(2, 5) VAR(2, 6) VAR(3, 4) VAR(4, 4) VAR(1, 6)
        dim3 g2((W + 511) / 512, (H + TR - 1) / TR, B);
        const size_t sm2 = (size_t)(TR / 4 + 3) * 2 * 131 * 4;
#define VAR2(U, MB) \
        cudaFuncSetAttribute(output_kernel<1, 1, 2, false, U, MB>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100000); \
        snprintf(nm, 64, "walker-staged PX2 U%d MINB%d TR=%d", U, MB, TR); \
        rep(nm, timeit([&] { output_kernel<1, 1, 2, false, U, MB><<<g2, 256, sm2>>>(op); }), bytes_k4);
        VAR2(2, 6) VAR2(4, 4) VAR2(2, 8)
    }
    for (int TR : {16, 32, 64}) {
        OutParams op{I, M, q, H, W, h, w, H, h, 0, 0, TR};
        dim3 g4((W + 1023) / 1024, (H + TR - 1) / TR, B);
        const size_t sm = (size_t)(TR / 4 + 3) * 2 * 259 * 4 + AsyncCfg<1, 1, 4>::RING_BYTES;
        cudaFuncSetAttribute(output_async_kernel<1, 1, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200000);
        int occ = 0; cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, output_async_kernel<1, 1, 4>, 256, sm);
        char nm[64];
        snprintf(nm, 64, "async-ring PX4 U8 TR=%d occ=%d", TR, occ);
        rep(nm, timeit([&] { output_async_kernel<1, 1, 4><<<g4, 256, sm>>>(op); }), bytes_k4);
    }
    {
        float* M1;
        CK(cudaMalloc(&M1, (size_t)2 * 2 * N * 4));
        OutParams op{I, M1, q, H, W, H, W, H, H, 0, 0, 64};
        dim3 g4((W + 1023) / 1024, (H + 63) / 64, 2);
        rep("walker-s1 PX4 (2 images)", timeit([&] { output_kernel<1, 1, 4, true><<<g4, 256>>>(op); }), 2.0 * (4.0 * N * 4));
        cudaFree(M1);
    }
    for (int TR : {32, 64}) {
        OutParams o{I, M, q, H, W, h, w, H, h, 0, 0, TR};
        const int nrl = TR / 4 + 3, ncl = 259;
        const size_t psm = 2 * (size_t)nrl * 2 * ncl * 4;
        auto k = output_persist_kernel<1, 1, 4>;
        cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)psm);
        int occ = 0; cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k, 256, psm);
        PersistParams pp{o, B, 4, sms * occ / 4, nrl, ncl};
        char nm[64];
        snprintf(nm, 64, "persist PX4 TR=%d occ=%d", TR, occ);
        rep(nm, timeit([&] { k<<<pp.ncb * pp.cpb, 256, psm>>>(pp); }), bytes_k4);
    }
    {
        using Cfg = TmaCfg<1, 1>;
        cudaFuncSetAttribute(output_tma_kernel<1, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Cfg::SMEM);
        for (int TR : {32, 64}) {
            TmaOutParams tp{I, M, q, H, W, h, w, B, TR, 4, sms / 4};
            char nm[64];
            snprintf(nm, 64, "tma persistent TR=%d", TR);
            rep(nm, timeit([&] { output_tma_kernel<1, 1><<<tp.ncb * tp.cpb, 256, Cfg::SMEM>>>(tp); }), bytes_k4);
        }
    }
    CK(cudaGetLastError());
    return 0;
}
