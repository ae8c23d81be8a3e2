// green_bench.cu -- experiment: SM-partitioned overlap of the low-res chain (K13) with the
// output pass (K4) through CUDA green contexts.  K13 is issue / shared-memory bound, K4 is
// HBM bound; running them concurrently on DISJOINT SM sets (chunk j+1's K13 while chunk j's
// K4 streams) can hide K13 under K4 if K4 still reaches the HBM rate on the smaller set.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o build/green_bench tools/green_bench.cu \
//        -Iinclude -Lpaper_1505_00996_b200 -lfgf -lcuda -Xlinker -rpath=$PWD/paper_1505_00996_b200
//   build/green_bench [batch]
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdio.h>
#include <stdlib.h>
#include <vector>
#include <algorithm>

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

struct Part {
    CUgreenCtx g[2];
    cudaStream_t s[2];
    int sms[2];
};

// Split the device's SMs into a group of (at least) n0 SMs and the remainder.
static bool make_part(CUdevice dev, int n0, Part& P) {
    CUdevResource all, grp[1], rest;
    CU(cuDeviceGetDevResource(dev, &all, CU_DEV_RESOURCE_TYPE_SM));
    unsigned ng = 1;
    if (cuDevSmResourceSplitByCount(grp, &ng, &all, &rest, 0, n0) != CUDA_SUCCESS || ng != 1)
        return false;
    CUdevResource* rs[2] = {&grp[0], &rest};
    for (int k = 0; k < 2; ++k) {
        CUdevResourceDesc d;
        CU(cuDevResourceGenerateDesc(&d, rs[k], 1));
        CU(cuGreenCtxCreate(&P.g[k], d, dev, CU_GREEN_CTX_DEFAULT_STREAM));
        CUstream cs;
        CU(cuGreenCtxStreamCreate(&cs, P.g[k], CU_STREAM_NON_BLOCKING, 0));
        P.s[k] = (cudaStream_t)cs;
        P.sms[k] = rs[k]->sm.smCount;
    }
    return true;
}

int main(int argc, char** argv) {
    const int B = argc > 1 ? atoi(argv[1]) : 256;
    const int H = 4096, W = 4096, r = 32, s = 4;
    const double eps = 0.01;
    const int h = H / s, w = W / s;
    const size_t N = (size_t)H * W, n = (size_t)h * w;
    CU(cuInit(0));
    CK(cudaSetDevice(0));
    CK(cudaFree(0));
    CUdevice dev;
    CU(cuDeviceGet(&dev, 0));
    float *I, *p, *q, *M;
    CK(cudaMalloc(&I, B * N * 4));
    CK(cudaMalloc(&p, B * N * 4));
    CK(cudaMalloc(&q, B * N * 4));
    CK(cudaMalloc(&M, B * 2 * n * 4));
    fill<<<1184, 256>>>(I, B * N, 1u);
    fill<<<1184, 256>>>(p, B * N, 2u);
    const size_t wsb = fgf_workspace_bytes(B, H, W, 1, 1, r, s);
    void* ws;
    CK(cudaMalloc(&ws, wsb));
    cudaStream_t main_s;
    CK(cudaStreamCreateWithFlags(&main_s, cudaStreamNonBlocking));
    CK(cudaDeviceSynchronize());
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    auto timeit = [&](auto&& body, int reps) {
        body();
        CK(cudaStreamSynchronize(main_s));
        CK(cudaDeviceSynchronize());
        std::vector<float> t;
        for (int i = 0; i < reps; ++i) {
            CK(cudaEventRecord(e0, main_s));
            body();
            CK(cudaEventRecord(e1, main_s));
            CK(cudaEventSynchronize(e1));
            float ms;
            CK(cudaEventElapsedTime(&ms, e0, e1));
            t.push_back(ms);
        }
        std::sort(t.begin(), t.end());
        return t[t.size() / 2];
    };
    // baseline: the library's whole filter
    float tb = timeit([&] { FG(fgf_filter_ws(I, p, q, B, H, W, 1, 1, r, eps, s, 0, ws, wsb, main_s)); }, 5);
    float tk13 = timeit([&] { FG(fgf_coefficients(I, p, M, B, H, W, 1, 1, r, eps, s, 0, ws, wsb, main_s)); }, 5);
    float tk4 = timeit([&] { FG(fgf_upsample_output(I, M, q, B, H, W, 1, 1, s, main_s)); }, 5);
    printf("baseline whole filter %.3f ms  K13 %.3f  K4 %.3f  (B=%d)\n", tb, tk13, tk4, B);
    fflush(stdout);

    const int splits[] = {48, 64, 72, 80, 88, 96, 104};
    std::vector<cudaEvent_t> ev(2 * B + 2);
    for (auto& e : ev) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    for (int n0 : splits) {
        Part P;
        if (!make_part(dev, n0, P)) { printf("split %d: failed\n", n0); continue; }
        // each stream alone on its partition
        auto on = [&](cudaStream_t st, auto&& f) {
            CK(cudaEventRecord(ev[0], main_s));
            CK(cudaStreamWaitEvent(st, ev[0], 0));
            f(st);
            CK(cudaEventRecord(ev[1], st));
            CK(cudaStreamWaitEvent(main_s, ev[1], 0));
        };
        float a13 = timeit([&] { on(P.s[0], [&](cudaStream_t st) {
            FG(fgf_coefficients(I, p, M, B, H, W, 1, 1, r, eps, s, 0, ws, wsb, st)); }); }, 3);
        float a4 = timeit([&] { on(P.s[1], [&](cudaStream_t st) {
            FG(fgf_upsample_output(I, M, q, B, H, W, 1, 1, s, st)); }); }, 3);
        float b4 = timeit([&] { on(P.s[0], [&](cudaStream_t st) {
            FG(fgf_upsample_output(I, M, q, B, H, W, 1, 1, s, st)); }); }, 3);
        printf("split %d/%d SMs: K13 on %d: %.3f ms | K4 on %d: %.3f ms | K4 on %d: %.3f ms\n",
               P.sms[0], P.sms[1], P.sms[0], a13, P.sms[1], a4, P.sms[0], b4);
        for (int c : {4, 8, 16, 32}) {
            if (c > B) continue;
            float tp = timeit([&] {
                CK(cudaEventRecord(ev[0], main_s));
                CK(cudaStreamWaitEvent(P.s[0], ev[0], 0));
                CK(cudaStreamWaitEvent(P.s[1], ev[0], 0));
                int j = 0;
                for (int b0 = 0; b0 < B; b0 += c, ++j) {
                    const int nb = std::min(c, B - b0);
                    FG(fgf_coefficients(I + b0 * N, p + b0 * N, M + b0 * 2 * n, nb, H, W, 1, 1, r,
                                        eps, s, 0, ws, wsb, P.s[0]));
                    CK(cudaEventRecord(ev[2 + j], P.s[0]));
                    CK(cudaStreamWaitEvent(P.s[1], ev[2 + j], 0));
                    FG(fgf_upsample_output(I + b0 * N, M + b0 * 2 * n, q + b0 * N, nb, H, W, 1, 1, s,
                                           P.s[1]));
                }
                CK(cudaEventRecord(ev[1], P.s[1]));
                CK(cudaStreamWaitEvent(main_s, ev[1], 0));
            }, 5);
            printf("  pipelined chunk %2d: %.3f ms  (%.0f Mpx/s)\n", c, tp, B * N / (tp * 1e3));
        }
        fflush(stdout);
        CK(cudaDeviceSynchronize());
        for (int k = 0; k < 2; ++k) {
            CK(cudaStreamDestroy(P.s[k]));
            CU(cuGreenCtxDestroy(P.g[k]));
        }
    }
    return 0;
}
