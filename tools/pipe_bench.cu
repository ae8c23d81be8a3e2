// Throughput microbenchmark of the instructions the low-res chain leans on (development tool):
// F2F.F64.F32, F2F.F32.F64, DADD, FADD, MUFU.RCP, integer bit ops.  Ops per clock per SM.
#include <cstdio>
#include <cstdint>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)
constexpr int ITER = 4096, ILP = 8;
__global__ void k_f2f64(const float* in, double* out) {
    float f[ILP]; double d[ILP];
    for (int i = 0; i < ILP; ++i) { f[i] = in[threadIdx.x + i]; d[i] = 0; }
    for (int it = 0; it < ITER; ++it) {
#pragma unroll
        for (int i = 0; i < ILP; ++i) { d[i] += (double)f[i]; f[i] = __int_as_float(__float_as_int(f[i]) ^ 1); }
    }
    double s = 0; for (int i = 0; i < ILP; ++i) s += d[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void k_dadd(const float* in, double* out) {
    double d[ILP], x = in[threadIdx.x];
    for (int i = 0; i < ILP; ++i) d[i] = in[i];
    for (int it = 0; it < ITER; ++it) {
#pragma unroll
        for (int i = 0; i < ILP; ++i) d[i] += x;
    }
    double s = 0; for (int i = 0; i < ILP; ++i) s += d[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void k_f2f32(const float* in, double* out) {
    double d[ILP]; float f[ILP];
    for (int i = 0; i < ILP; ++i) { d[i] = in[threadIdx.x + i]; f[i] = 0; }
    for (int it = 0; it < ITER; ++it) {
#pragma unroll
        for (int i = 0; i < ILP; ++i) { f[i] += (float)d[i]; }
    }
    double s = 0; for (int i = 0; i < ILP; ++i) s += f[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void k_rcp(const float* in, double* out) {
    float f[ILP];
    for (int i = 0; i < ILP; ++i) f[i] = in[threadIdx.x + i] + 1.5f;
    for (int it = 0; it < ITER; ++it) {
#pragma unroll
        for (int i = 0; i < ILP; ++i) f[i] = __frcp_rn(f[i]) + 0.5f;
    }
    double s = 0; for (int i = 0; i < ILP; ++i) s += f[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void k_rcpapprox(const float* in, double* out) {
    float f[ILP];
    for (int i = 0; i < ILP; ++i) f[i] = in[threadIdx.x + i] + 1.5f;
    for (int it = 0; it < ITER; ++it) {
#pragma unroll
        for (int i = 0; i < ILP; ++i) { float r; asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(f[i])); f[i] = r + 0.5f; }
    }
    double s = 0; for (int i = 0; i < ILP; ++i) s += f[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void k_fadd(const float* in, double* out) {
    float d[ILP], x = in[threadIdx.x];
    for (int i = 0; i < ILP; ++i) d[i] = in[i];
    for (int it = 0; it < ITER; ++it) {
#pragma unroll
        for (int i = 0; i < ILP; ++i) d[i] += x;
    }
    double s = 0; for (int i = 0; i < ILP; ++i) s += d[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
// exact float -> double by integer bit manipulation (normal numbers and zero)
__device__ __forceinline__ double f2d_bits(float f) {
    const uint32_t u = __float_as_uint(f);
    const uint32_t hi = ((u & 0x7fffffffu) >> 3) + 0x38000000u;
    const uint32_t h2 = (u & 0x7f800000u) ? (hi | (u & 0x80000000u)) : (u & 0x80000000u);
    return __hiloint2double((int)h2, (int)(u << 29));
}
__global__ void k_f2dbits(const float* in, double* out) {
    float f[ILP]; double d[ILP];
    for (int i = 0; i < ILP; ++i) { f[i] = in[threadIdx.x + i]; d[i] = 0; }
    for (int it = 0; it < ITER; ++it) {
#pragma unroll
        for (int i = 0; i < ILP; ++i) { d[i] += f2d_bits(f[i]); f[i] = __int_as_float(__float_as_int(f[i]) ^ 1); }
    }
    double s = 0; for (int i = 0; i < ILP; ++i) s += d[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
template <typename K>
int run(const char* nm, K k, const float* in, double* out, int per_iter_ops) {
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    dim3 grid(sms * 4), block(512);
    k<<<grid, block>>>(in, out);
    CK(cudaDeviceSynchronize());
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    cudaEventRecord(a); k<<<grid, block>>>(in, out); cudaEventRecord(b); CK(cudaEventSynchronize(b));
    float ms; cudaEventElapsedTime(&ms, a, b);
    double ops = (double)grid.x * block.x * ITER * ILP * per_iter_ops;
    double per_clk_sm = ops / (ms * 1e-3) / sms / (clk * 1e3);
    printf("%-22s %8.3f ms  %7.1f ops/clk/SM (at %d MHz nominal)\n", nm, ms, per_clk_sm, clk / 1000);
    return 0;
}
int main() {
    float* in; double* out;
    CK(cudaMalloc(&in, 1 << 20)); CK(cudaMemset(in, 0, 1 << 20));
    CK(cudaMalloc(&out, 64 << 20));
    run("F2F.F64.F32 (+DADD)", k_f2f64, in, out, 1);
    run("f2d bits (+DADD)", k_f2dbits, in, out, 1);
    run("DADD", k_dadd, in, out, 1);
    run("F2F.F32.F64 (+FADD)", k_f2f32, in, out, 1);
    run("FADD", k_fadd, in, out, 1);
    run("rcp_rn (+FADD)", k_rcp, in, out, 1);
    run("rcp.approx (+FADD)", k_rcpapprox, in, out, 1);
    return 0;
}
