// colour_pipe_bench.cu -- experiment: config 3 (64 x 1920x1080, C_I = C_p = 3, r = 8, s = 4
// block mean) as a three-stream chunk pipeline of the public stage calls: K0 block means of
// chunk j+1 (HBM bound) || K1 + K3 low-res chain of chunk j (issue bound) || K4 of chunk j-1
// (HBM bound), optionally with the low-res chain on its own green-context SM partition.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++17 -o build/colour_pipe_bench \
//        tools/colour_pipe_bench.cu -Iinclude -Lpaper_1505_00996_b200 -lfgf -lcuda \
//        -Xlinker -rpath='$ORIGIN/../paper_1505_00996_b200'
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdio.h>
#include <stdlib.h>
#include <math.h>
#include <algorithm>
#include <vector>

#include "fgf.h"

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { \
    fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); exit(1); } } while (0)
#define CU(x) do { CUresult e_ = (x); if (e_ != CUDA_SUCCESS) { const char* s_; \
    cuGetErrorString(e_, &s_); fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, s_); exit(1); } } while (0)
#define FG(x) do { int e_ = (x); if (e_ != 0) { \
    fprintf(stderr, "%s:%d fgf %s\n", __FILE__, __LINE__, fgf_status_str(e_)); exit(1); } } while (0)

__global__ void fill(float* x, size_t n, unsigned seed) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n;
         i += (size_t)gridDim.x * blockDim.x) {
        unsigned v = (unsigned)i * 2654435761u ^ seed;
        v ^= v >> 13; v *= 0x5bd1e995u; v ^= v >> 15;
        x[i] = (v & 0xffffff) * (1.0f / 16777216.0f);
    }
}
__global__ void maxdiff(const float* a, const float* b, size_t n, float* out) {
    float m = 0.f;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n;
         i += (size_t)gridDim.x * blockDim.x) m = fmaxf(m, fabsf(a[i] - b[i]));
    atomicMax(reinterpret_cast<int*>(out), __float_as_int(m));
}

int main(int argc, char** argv) {
    const int B = argc > 1 ? atoi(argv[1]) : 64;
    const int H = 1080, W = 1920, CI = 3, CP = 3, r = 8, s = 4, sub = FGF_SUB_BILINEAR;
    const double eps = 0.01;
    const int h = (H + s - 1) / s, w = (W + s - 1) / s, rl = 2;
    const size_t N = (size_t)H * W, n = (size_t)h * w;
    const int NC = (CI + 1) * CP;
    CU(cuInit(0));
    CK(cudaSetDevice(0));
    CK(cudaFree(0));
    CUdevice dev;
    CU(cuDeviceGet(&dev, 0));
    float *I, *p, *q, *q0, *Is, *ps, *M, *dm;
    CK(cudaMalloc(&I, B * CI * N * 4));
    CK(cudaMalloc(&p, B * CP * N * 4));
    CK(cudaMalloc(&q, B * CP * N * 4));
    CK(cudaMalloc(&q0, B * CP * N * 4));
    CK(cudaMalloc(&Is, B * CI * n * 4));
    CK(cudaMalloc(&ps, B * CP * n * 4));
    CK(cudaMalloc(&M, B * NC * n * 4));
    CK(cudaMalloc(&dm, 4));
    fill<<<1184, 256>>>(I, B * CI * N, 1u);
    fill<<<1184, 256>>>(p, B * CP * N, 2u);
    const size_t wsb = fgf_workspace_bytes(B, H, W, CI, CP, r, s);
    const size_t lwsb = fgf_lowres_workspace_bytes(B, h, w, CI, CP);
    void *ws, *lws;
    CK(cudaMalloc(&ws, wsb));
    CK(cudaMalloc(&lws, lwsb));
    cudaStream_t ms, sa, sb, sc;
    CK(cudaStreamCreateWithFlags(&ms, cudaStreamNonBlocking));
    CK(cudaStreamCreateWithFlags(&sa, cudaStreamNonBlocking));
    CK(cudaStreamCreateWithFlags(&sb, cudaStreamNonBlocking));
    CK(cudaStreamCreateWithFlags(&sc, cudaStreamNonBlocking));
    CK(cudaDeviceSynchronize());
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    std::vector<cudaEvent_t> ev(4 * B + 8);
    for (auto& e : ev) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    auto timeit = [&](auto&& body, int reps) {
        body();
        CK(cudaDeviceSynchronize());
        std::vector<float> t;
        for (int i = 0; i < reps; ++i) {
            CK(cudaEventRecord(e0, ms));
            body();
            CK(cudaEventRecord(e1, ms));
            CK(cudaEventSynchronize(e1));
            float x;
            CK(cudaEventElapsedTime(&x, e0, e1));
            t.push_back(x);
        }
        std::sort(t.begin(), t.end());
        return t[t.size() / 2];
    };
    auto check = [&](const char* what) {
        CK(cudaMemset(dm, 0, 4));
        maxdiff<<<1184, 256>>>(q, q0, B * CP * N, dm);
        float d;
        CK(cudaMemcpy(&d, dm, 4, cudaMemcpyDeviceToHost));
        printf("    %s max|q - q_lib| = %g\n", what, d);
    };
    float tb = timeit([&] { FG(fgf_filter_ws(I, p, q0, B, H, W, CI, CP, r, eps, s, sub, ws, wsb, ms)); }, 7);
    printf("library whole filter: %.3f ms (B=%d)\n", tb, B);
    auto stages = [&](int b0, int nb, cudaStream_t s0, cudaStream_t s1, cudaStream_t s2, int j) {
        FG(fgf_subsample(I + b0 * CI * N, Is + b0 * CI * n, nb * CI, H, W, s, sub, s0));
        FG(fgf_subsample(p + b0 * CP * N, ps + b0 * CP * n, nb * CP, H, W, s, sub, s0));
        if (s1 != s0) {
            CK(cudaEventRecord(ev[8 + 2 * j], s0));
            CK(cudaStreamWaitEvent(s1, ev[8 + 2 * j], 0));
        }
        FG(fgf_lowres_mean(Is + b0 * CI * n, ps + b0 * CP * n, M + b0 * NC * n, nb, h, w, CI, CP,
                           rl, eps, lws, lwsb, s1));
        if (s2 != s1) {
            CK(cudaEventRecord(ev[9 + 2 * j], s1));
            CK(cudaStreamWaitEvent(s2, ev[9 + 2 * j], 0));
        }
        FG(fgf_upsample_output(I + b0 * CI * N, M + b0 * NC * n, q + b0 * CP * N, nb, H, W, CI, CP,
                               s, s2));
    };
    float ts = timeit([&] { stages(0, B, ms, ms, ms, 0); }, 7);
    printf("stage calls, one stream: %.3f ms\n", ts);
    check("sequential");
    float tk0 = timeit([&] {
        FG(fgf_subsample(I, Is, B * CI, H, W, s, sub, ms));
        FG(fgf_subsample(p, ps, B * CP, H, W, s, sub, ms)); }, 7);
    float tlr = timeit([&] {
        FG(fgf_lowres_mean(Is, ps, M, B, h, w, CI, CP, rl, eps, lws, lwsb, ms)); }, 7);
    float tk4 = timeit([&] { FG(fgf_upsample_output(I, M, q, B, H, W, CI, CP, s, ms)); }, 7);
    printf("K0 x2 %.3f | K1+K3 %.3f | K4 %.3f ms\n", tk0, tlr, tk4);

    auto pipe = [&](int c, cudaStream_t A, cudaStream_t Bs, cudaStream_t C) {
        CK(cudaEventRecord(ev[0], ms));
        CK(cudaStreamWaitEvent(A, ev[0], 0));
        CK(cudaStreamWaitEvent(Bs, ev[0], 0));
        CK(cudaStreamWaitEvent(C, ev[0], 0));
        int j = 0;
        for (int b0 = 0; b0 < B; b0 += c, ++j) stages(b0, std::min(c, B - b0), A, Bs, C, j);
        CK(cudaEventRecord(ev[1], C));
        CK(cudaStreamWaitEvent(ms, ev[1], 0));
        CK(cudaEventRecord(ev[2], A));
        CK(cudaStreamWaitEvent(ms, ev[2], 0));
        CK(cudaEventRecord(ev[3], Bs));
        CK(cudaStreamWaitEvent(ms, ev[3], 0));
    };
    for (int c : {2, 4, 8, 16, 32}) {
        float tp = timeit([&] { pipe(c, sa, sb, sc); }, 7);
        printf("3-stream pipeline, chunk %2d: %.3f ms\n", c, tp);
    }
    check("pipelined");
    // K0 and K4 share one stream (both HBM bound), the low-res chain on the other
    for (int c : {4, 8, 16}) {
        float tp = timeit([&] { pipe(c, sa, sb, sa); }, 7);
        printf("2-stream (K0,K4 | K1+K3), chunk %2d: %.3f ms\n", c, tp);
    }
    // green partitions: the low-res chain on n0 SMs, K0 / K4 on the rest
    for (int n0 : {24, 40, 56, 72}) {
        CUdevResource all, grp[1], rest;
        CU(cuDeviceGetDevResource(dev, &all, CU_DEV_RESOURCE_TYPE_SM));
        unsigned ng = 1;
        if (cuDevSmResourceSplitByCount(grp, &ng, &all, &rest, 0, n0) != CUDA_SUCCESS) continue;
        CUdevResource* rs[2] = {&grp[0], &rest};
        CUgreenCtx g[2];
        cudaStream_t gs[2];
        for (int k = 0; k < 2; ++k) {
            CUdevResourceDesc d;
            CU(cuDevResourceGenerateDesc(&d, rs[k], 1));
            CU(cuGreenCtxCreate(&g[k], d, dev, CU_GREEN_CTX_DEFAULT_STREAM));
            CUstream cs;
            CU(cuGreenCtxStreamCreate(&cs, g[k], CU_STREAM_NON_BLOCKING, 0));
            gs[k] = (cudaStream_t)cs;
        }
        cudaStream_t gs2;
        {
            CUstream cs;
            CU(cuGreenCtxStreamCreate(&cs, g[1], CU_STREAM_NON_BLOCKING, 0));
            gs2 = (cudaStream_t)cs;
        }
        for (int c : {4, 8, 16}) {
            float tp = timeit([&] { pipe(c, gs[1], gs[0], gs2); }, 7);
            printf("green %d/%d SMs (K1+K3 | K0, K4 on 2 streams), chunk %2d: %.3f ms\n",
                   grp[0].sm.smCount, rest.sm.smCount, c, tp);
        }
        CK(cudaDeviceSynchronize());
        CK(cudaStreamDestroy(gs[0]));
        CK(cudaStreamDestroy(gs[1]));
        CK(cudaStreamDestroy(gs2));
        CU(cuGreenCtxDestroy(g[0]));
        CU(cuGreenCtxDestroy(g[1]));
    }
    check("green");
    return 0;
}
