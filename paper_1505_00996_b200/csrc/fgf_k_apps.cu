// fgf_k_apps.cu -- application kernels around the filter:
//   luma  SPEC to_grayscale: L = 0.299 R + 0.587 G + 0.114 B of a planar RGB image,
//         the shared gray guidance of SPEC's enhance;
//   blend out = gain x img + (1 - gain) x q, i.e. (img - q) gain + q (Fig. 2 caption),
//         in place on q, for guidance other than the image itself (where the gain folds into
//         the mean maps instead, fgf_enhance_ws).
#include "fgf_host.cuh"

namespace fgf {

// grid (ceil(HW / (256 x 4)), batch), block 256: 4 pixels per thread.
__global__ void __launch_bounds__(256) luma_kernel(const float* __restrict__ img,
                                                   float* __restrict__ L, size_t N) {
    const size_t b = blockIdx.y;
    const float* R = img + b * 3 * N;
    const float* G = R + N;
    const float* B = G + N;
    float* o = L + b * N;
    for (size_t i = ((size_t)blockIdx.x * 256 + threadIdx.x) * 4, k = 0; k < 4 && i < N; ++i, ++k)
        o[i] = fmaf(0.114f, __ldg(B + i), fmaf(0.587f, __ldg(G + i), 0.299f * __ldg(R + i)));
}

// grid (ceil(n / (256 x 4))), block 256.
__global__ void __launch_bounds__(256) blend_kernel(const float* __restrict__ img,
                                                    float* __restrict__ q, size_t n, float k0,
                                                    float k1) {
    for (size_t i = ((size_t)blockIdx.x * 256 + threadIdx.x) * 4, k = 0; k < 4 && i < n; ++i, ++k)
        q[i] = fmaf(k1, q[i], k0 * __ldg(img + i));
}

int launch_luma(const float* img, float* L, int batch, size_t N, cudaStream_t st) {
    dim3 grid((unsigned)((N + 1023) / 1024), batch);
    ProfScope ps(KIND_SUB, st);
    luma_kernel<<<grid, 256, 0, st>>>(img, L, N);
    ++g_last_launches;
    return last_error();
}

int launch_blend(const float* img, float* q, size_t n, double gain, cudaStream_t st) {
    dim3 grid((unsigned)((n + 1023) / 1024));
    ProfScope ps(KIND_OUT, st);
    blend_kernel<<<grid, 256, 0, st>>>(img, q, n, (float)gain, (float)(1.0 - gain));
    ++g_last_launches;
    return last_error();
}

}  // namespace fgf
