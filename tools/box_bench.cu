// Microbenchmark of the low-res box kernels (K1 statistics, K3 box of a, b) on
// config-4-shaped low-res data (B x 1024^2, r' = 8).  Development tool, not product code.
#include <cstdio>
#include <cstdlib>
#include <algorithm>
#include "../paper_1505_00996_b200/csrc/fgf_kernels.cuh"
using namespace fgf;
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); exit(1); } } while (0)
template <typename F> float timeit(F f, int reps = 5) {
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    f(); CK(cudaDeviceSynchronize());
    cudaEventRecord(a); for (int r = 0; r < reps; ++r) f(); cudaEventRecord(b);
    CK(cudaEventSynchronize(b)); float ms; cudaEventElapsedTime(&ms, a, b); return ms / reps;
}
template <int MODE, int G, int MINB, int NT = 256>
void run(const char* nm, StripParams sp, int B, int TH) {
    using C = StripConfig<MODE, 1, 1, NT, G, MINB>;
    sp.TW = NT - 2 * sp.R; sp.TH = TH; sp.VP = NT + 2 * sp.R + C::K + 1;
    size_t smem = C::smem(sp.VP);
    auto k = box_strip_kernel<MODE, 1, 1, NT, G, MINB>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    int strips = (sp.w + sp.TW - 1) / sp.TW;
    dim3 grid(strips, (sp.h + TH - 1) / TH, B);
    int occ = 0; cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k, NT, smem);
    float ms = timeit([&] { k<<<grid, NT, smem>>>(sp); });
    printf("%-10s G=%d MINB=%d TH=%3d smem=%6zu occ=%d grid=%6d  %8.3f ms  %6.2f us/img\n", nm, G, MINB, TH, smem, occ, grid.x * grid.y * grid.z, ms, 1e3 * ms / B);
    CK(cudaGetLastError());
}
int main(int argc, char** argv) {
    const int B = argc > 1 ? atoi(argv[1]) : 64;
    const int h = 1024, w = 1024, R = 8;
    const size_t n = (size_t)h * w;
    float *Is, *ps, *ab, *mab;
    CK(cudaMalloc(&Is, B * n * 4)); CK(cudaMalloc(&ps, B * n * 4));
    CK(cudaMalloc(&ab, B * 2 * n * 4)); CK(cudaMalloc(&mab, B * 2 * n * 4));
    CK(cudaMemset(Is, 0, B * n * 4)); CK(cudaMemset(ps, 0, B * n * 4)); CK(cudaMemset(ab, 0, B * 2 * n * 4));
    StripParams st{}; st.srcI = Is; st.srcP = ps; st.imgI = n; st.imgP = n; st.planeI = n; st.planeP = n;
    st.row = w; st.col = 1; st.dst = ab; st.h = h; st.w = w; st.R = R; st.eps = 0.01;
    StripParams mp{}; mp.srcI = ab; mp.srcP = ab; mp.imgI = 2 * n; mp.imgP = 0; mp.planeI = n; mp.planeP = 0;
    mp.row = w; mp.col = 1; mp.dst = mab; mp.h = h; mp.w = w; mp.R = R; mp.eps = 0.01;
    for (int TH : {16, 32, 64}) {
        run<MODE_STATS, 8, 2>("stats", st, B, TH);
        run<MODE_STATS, 4, 2>("stats", st, B, TH);
        run<MODE_STATS, 4, 3>("stats", st, B, TH);
        run<MODE_STATS, 4, 4>("stats", st, B, TH);
        run<MODE_STATS, 2, 4>("stats", st, B, TH);
        run<MODE_MEAN, 8, 2>("mean", mp, B, TH);
        run<MODE_MEAN, 4, 4>("mean", mp, B, TH);
        run<MODE_MEAN, 2, 4>("mean", mp, B, TH);
    }
    return 0;
}
