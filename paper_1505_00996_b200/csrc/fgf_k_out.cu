// fgf_k_out.cu -- K4: bilinear upsampling of mean_a, mean_b and q = mean_a * I + mean_b
// (Alg. 2 steps 6-7), launch geometry and variant choice.
#include "fgf_host.cuh"

namespace fgf {

// Largest low-res rectangle (rows x cols) a CTA of TR rows and `cols` pixels touches (R5).
int lowres_span(int T, int n_dst, int n_src) {
    auto lo = [&](int d) {
        long long num = (long long)(2 * d + 1) * n_src - n_dst;
        if (num <= 0) return 0;
        long long q = num / (2LL * n_dst);
        return (int)std::min<long long>(q, n_src - 1);
    };
    int best = 1;
    for (int d0 = 0; d0 < n_dst; d0 += T) {
        int dl = std::min(n_dst, d0 + T) - 1;
        best = std::max(best, std::min(lo(dl) + 1, n_src - 1) - lo(d0) + 1);
    }
    return best;
}

// Columns of the staged rectangle: the span from a 4-aligned origin, rounded up to 4.
int lowres_cols(int T, int n_dst, int n_src) { return (lowres_span(T, n_dst, n_src) + 6) & ~3; }

constexpr size_t kOutSmemBudget = 44 * 1024;

template <int CI, int CP, int PX, typename E = float>
int launch_output_px(const OutParams& op0, int images, const Plan& P, cudaStream_t st) {
    constexpr int NC = (CI + 1) * CP;
    OutParams op = op0;
    const bool s1 = op.hg == op.Hg && P.w == P.W;
    size_t smem = 0;
    if (s1) {
        op.TR = 64;
    } else {
        const int ncl = lowres_cols(256 * PX, P.W, P.w);
        op.TR = 8;
        for (int tr = kMaxTR; tr >= 8; tr /= 2) {
            const size_t b = (size_t)lowres_span(tr, op.Hg, op.hg) * NC * ncl * sizeof(float);
            if (b <= kOutSmemBudget) { op.TR = tr; break; }
        }
        // small launches (single images): shorter bands until ~2 waves of 4 CTAs per SM exist
        const long long ncb = (P.W + 256 * PX - 1) / (256 * PX);
        while (op.TR > 8 && ncb * ((P.H + op.TR - 1) / op.TR) * images < 2LL * 4 * 148) op.TR /= 2;
        if (const char* e = dev_env("FGF_K4_TR")) {      // development knob: band height
            const int tr = atoi(e);
            if (tr >= 1 && tr <= op.TR) op.TR = tr;
        }
        smem = (size_t)lowres_span(op.TR, op.Hg, op.hg) * NC * ncl * sizeof(float);
        if (smem > 200 * 1024) return FGF_ERR_UNSUPPORTED;
        // optional floor on the dynamic smem: caps K4 CTAs/SM so the low-res stream's CTAs
        // can be co-resident (experiment knob)
        if (const char* e = dev_env("FGF_K4_SMEM_MIN")) smem = std::max<size_t>(smem, (size_t)atoi(e));
    }
    dim3 grid((P.W + 256 * PX - 1) / (256 * PX), (P.H + op.TR - 1) / op.TR, images);
    if constexpr (PX * sizeof(E) >= 4) {   // cp.async moves 4, 8 or 16 bytes
        if (!s1 && dev_env("FGF_NO_ASYNC") == nullptr) {
            // cp.async ring variant: prefetch held in shared memory, not registers
            const size_t asm_ = smem + AsyncCfg<CI, CP, PX, E>::RING_BYTES;
            if (asm_ <= 200 * 1024) {
                auto kern = output_async_kernel<CI, CP, PX, E>;
                set_smem(kern, asm_);
                ProfScope ps(KIND_OUT, st);
                if (op.pdl) {
                    cudaLaunchConfig_t cfg = {};
                    cfg.gridDim = grid;
                    cfg.blockDim = dim3(256);
                    cfg.dynamicSmemBytes = asm_;
                    cfg.stream = st;
                    cudaLaunchAttribute at[1];
                    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
                    at[0].val.programmaticStreamSerializationAllowed = 1;
                    cfg.attrs = at;
                    cfg.numAttrs = 1;
                    if (cudaLaunchKernelEx(&cfg, kern, op) != cudaSuccess) return FGF_ERR_CUDA;
                } else {
                    kern<<<grid, 256, asm_, st>>>(op);
                }
                ++g_last_launches;
                return last_error();
            }
        }
    }
    if constexpr (PX * sizeof(float) > 16) {
        return FGF_ERR_UNSUPPORTED;   // the register walker moves fp32 map vectors of PX
    } else {
        ProfScope ps(KIND_OUT, st);
        if (s1) {
            output_kernel<CI, CP, PX, true, 0, 0, 0, E><<<grid, 256, 0, st>>>(op);
        } else {
            auto kern = output_kernel<CI, CP, PX, false, 0, 0, 0, E>;
            set_smem(kern, smem);
            kern<<<grid, 256, smem, st>>>(op);
        }
        ++g_last_launches;
        return last_error();
    }
}

// Colour guidance with several p channels, fp32, 4-pixel alignment: the channel-split K4
// (opt-in, FGF_K4_SPLIT=1: measured 0.84 ms vs 0.76 ms for the per-pixel walker on config 3).
template <int CI, int CP>
int launch_output_split(const OutParams& op0, int images, const Plan& P, cudaStream_t st) {
    using C = SplitCfg<CI, CP>;
    constexpr int NC = C::NC;
    OutParams op = op0;
    const int ncl = lowres_cols(64 * C::PX, P.W, P.w);
    op.TR = 8;
    for (int tr = kMaxTR; tr >= 8; tr /= 2) {
        const size_t b = (size_t)lowres_span(tr, op.Hg, op.hg) * NC * ncl * sizeof(float);
        if (b <= kOutSmemBudget) { op.TR = tr; break; }
    }
    const long long ncb = (P.W + 64 * C::PX - 1) / (64 * C::PX);
    while (op.TR > 8 && ncb * ((P.H + op.TR - 1) / op.TR) * images < 2LL * 3 * 148) op.TR /= 2;
    const size_t smem = (size_t)lowres_span(op.TR, op.Hg, op.hg) * NC * ncl * sizeof(float) +
                        C::RING_BYTES + C::BAR_BYTES;
    if (smem > 200 * 1024) return FGF_ERR_UNSUPPORTED;
    dim3 grid((unsigned)ncb, (P.H + op.TR - 1) / op.TR, images);
    auto kern = output_split_kernel<CI, CP>;
    set_smem(kern, smem);
    ProfScope ps(KIND_OUT, st);
    kern<<<grid, C::NT, smem, st>>>(op);
    ++g_last_launches;
    return last_error();
}

// Pixels per thread: as wide as alignment allows while the coefficient registers fit.
template <int CI, int CP, typename E = float>
int launch_output_t(const OutParams& op, int images, const Plan& P, cudaStream_t st) {
    constexpr int NC = (CI + 1) * CP;
    if constexpr (CI == 3 && CP >= 2 && sizeof(E) == 4) {
        const uintptr_t al = reinterpret_cast<uintptr_t>(op.I) | reinterpret_cast<uintptr_t>(op.q);
        const bool s1 = op.hg == op.Hg && P.w == P.W;
        if (!s1 && P.W % 4 == 0 && (al & 15u) == 0 && dev_env("FGF_K4_SPLIT") != nullptr) {
            const int rc = launch_output_split<CI, CP>(op, images, P, st);
            if (rc != FGF_ERR_UNSUPPORTED) return rc;
        }
    }
    constexpr uintptr_t ES = sizeof(E);
    const uintptr_t ai = reinterpret_cast<uintptr_t>(op.I) | reinterpret_cast<uintptr_t>(op.q);
    const uintptr_t am = reinterpret_cast<uintptr_t>(op.M);
    if constexpr (ES == 1) {   // 8-bit codes: 8 pixels (8 bytes) per thread and row
        const bool s1 = op.hg == op.Hg && P.w == P.W;
        if (NC <= 2 && !s1 && P.W % 8 == 0 && (ai & 7u) == 0 && (am & 15u) == 0 &&
            dev_env("FGF_K4_U8PX4") == nullptr) {
            const int rc = launch_output_px<CI, CP, (NC <= 2 ? 8 : 1), E>(op, images, P, st);
            if (rc != FGF_ERR_UNSUPPORTED) return rc;
        }
    }
    if (NC <= 2 && P.W % 4 == 0 && (ai & (4 * ES - 1)) == 0 && (am & 15u) == 0)
        return launch_output_px<CI, CP, (NC <= 2 ? 4 : 1), E>(op, images, P, st);
    if constexpr (NC > 4 && ES == 4) {
        // colour, fp32: 2 pixels per thread (config 3 K4 0.708 -> 0.668 ms; FGF_K4_PX1=1: one)
        if (dev_env("FGF_K4_PX1") == nullptr && P.W % 2 == 0 && (ai & 7u) == 0 && (am & 7u) == 0)
            return launch_output_px<CI, CP, 2, E>(op, images, P, st);
    }
    if (NC <= 4 && P.W % 2 == 0 && (ai & (2 * ES - 1)) == 0 && (am & 7u) == 0)
        return launch_output_px<CI, CP, (NC <= 4 ? 2 : 1), E>(op, images, P, st);
    return launch_output_px<CI, CP, 1, E>(op, images, P, st);
}

int launch_output(const void* I, const float* M, void* q, int images, const Plan& P,
                  cudaStream_t st, const Band* band) {
    const Band b = band ? *band : Band{P.H, P.h, 0, 0, P.h};
    OutParams op{I, M, q, P.H, P.W, b.hm, P.w, b.Hg, b.hg, b.Yoff, b.yoff, P.TR, P.pdl_out ? 1 : 0};
    if (P.dtype != FGF_F32) {
        // reduced-precision I/O: gray -> gray, colour -> colour, colour guide -> one channel
        const int key = P.CI * 10 + P.CP;
        if (P.dtype == FGF_U8) {
            if (key == 11) return launch_output_t<1, 1, unsigned char>(op, images, P, st);
            if (key == 31) return launch_output_t<3, 1, unsigned char>(op, images, P, st);
            if (key == 33) return launch_output_t<3, 3, unsigned char>(op, images, P, st);
        } else if (P.dtype == FGF_F16) {
            if (key == 11) return launch_output_t<1, 1, __half>(op, images, P, st);
            if (key == 31) return launch_output_t<3, 1, __half>(op, images, P, st);
            if (key == 33) return launch_output_t<3, 3, __half>(op, images, P, st);
        } else {
            if (key == 11) return launch_output_t<1, 1, __nv_bfloat16>(op, images, P, st);
            if (key == 31) return launch_output_t<3, 1, __nv_bfloat16>(op, images, P, st);
            if (key == 33) return launch_output_t<3, 3, __nv_bfloat16>(op, images, P, st);
        }
        return FGF_ERR_UNSUPPORTED;
    }
    switch (P.CI * 10 + P.CP) {
        case 11: return launch_output_t<1, 1>(op, images, P, st);
        case 12: return launch_output_t<1, 2>(op, images, P, st);
        case 13: return launch_output_t<1, 3>(op, images, P, st);
        case 14: return launch_output_t<1, 4>(op, images, P, st);
        case 31: return launch_output_t<3, 1>(op, images, P, st);
        case 32: return launch_output_t<3, 2>(op, images, P, st);
        case 33: return launch_output_t<3, 3>(op, images, P, st);
        case 34: return launch_output_t<3, 4>(op, images, P, st);
    }
    return FGF_ERR_SHAPE;
}

}  // namespace fgf
