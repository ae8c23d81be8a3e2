/*
 * fgf.h -- C ABI of the B200-native Fast Guided Filter library (libfgf.so).
 *
 * The operation is Algorithm 2 of K. He, J. Sun, "Fast Guided Filter" (arXiv 1505.00996),
 * PAPER.md P:67-88 (citation keys: P:n = PAPER.md line n, S:n = SPEC.md line n, Rn = the
 * reading n listed in DESIGN.md "Readings"):
 *
 *   I' = f_subsample(I, s), p' = f_subsample(p, s), r' = r/s
 *   mean_I, mean_p, corr_I, corr_Ip = f_mean(., r') of I', p', I'.*I', I'.*p'
 *   var_I = corr_I - mean_I^2, cov_Ip = corr_Ip - mean_I mean_p
 *   a = cov_Ip / (var_I + eps), b = mean_p - a mean_I                  (Eq.2-3)
 *   mean_a = f_mean(a, r'), mean_b = f_mean(b, r')
 *   q = f_upsample(mean_a, s) .* I + f_upsample(mean_b, s), I at FULL resolution
 *
 * with I the guidance, p the filtering input and q the output.  A 3-channel
 * guidance uses the 3x3 ridge-regression solve a = (Sigma + eps U)^-1 (corr_Ip - mu p_bar),
 * b = p_bar - a^T mu, q = mean_a^T I + mean_b (R9; the cited journal version).
 *
 * Conventions fixed where the paper is silent:
 *   R1 f_mean clips the (2r'+1)^2 window to the image and divides by the in-bounds count
 *   R2 r' = max(1, floor(r/s + 1/2));  R6 low-res size h = ceil(H/s), w = ceil(W/s)
 *   R3 FGF_SUB_NEAREST takes I[y*s][x*s];  R4 FGF_SUB_BILINEAR is the clipped s x s block mean
 *   R5 bilinear upsampling maps x -> (x + 1/2) * w/W - 1/2, clamped to [0, w-1]
 *   R8 gray: var_I < 0 is clamped to 0;  R11 q is not clamped
 *
 * LAYOUT.  Every image buffer is dense, planar, row-major fp32: [batch][C][H][W]; I has
 * C_I channels, p and q have C_p channels.  Offsets are computed in 64-bit.
 *
 * OWNERSHIP.  The caller owns I, p, q and any workspace; the library never frees caller
 * memory.  fgf_filter() keeps one internal grow-only workspace per device (freed at exit).
 *
 * SYNCHRONISATION.  Device-pointer entry points validate synchronously on the host, before
 * any launch, then enqueue kernels on the given stream and return without synchronising.
 * Launch failures return FGF_ERR_CUDA; asynchronous faults surface at the caller's next
 * synchronisation (with FGF_DEBUG_SYNC=1 in the environment every launch is followed by a
 * device synchronisation and the faulting call returns FGF_ERR_CUDA).  Every launch is wrapped
 * in an NVTX range named after its kernel.  After any non-OK status q is unspecified.  fgf_filter_host() is
 * synchronous: it returns when q is in host memory.
 *
 * REENTRANCY.  Calls with distinct workspaces and streams are thread-safe.  Results are
 * deterministic (no atomics; fixed reduction order) and independent of batch size and of
 * how a batch is split across calls or devices.
 *
 * PRECISION.  fp32 storage; box statistics, var/cov and the 3x3 solve in fp64; a, b stored
 * in fp32; the box of a, b accumulated in fp64 (colour guidance; gray guidance at s = 1 and
 * for wide windows, engine K5) or fp32 (gray guidance in K13, R17, at most 512
 * running steps per segment); upsample + output in fp32.
 *
 * ENGINES (one choice per call, fixed by the arguments): gray guidance at s = 1
 * runs the exact guided filter (Alg. 1) as ONE kernel (K5) for r >= 4; gray guidance at s > 1
 * runs K13 (r' <= 12) or K5 (wider r'), then K4; colour guidance runs K0/K1/K3 then K4.
 *
 * GRAPH CACHE.  fgf_filter_ws / fgf_filter_ex_ws calls of at most 32 Mi output pixels on a
 * non-default stream are recorded on their first occurrence and, when the same arguments
 * (pointers, sizes, parameters, workspace, stream) occur again, captured into a CUDA graph and
 * replayed from then on (no per-launch host cost, no validation queries: the caller keeps the
 * buffers valid, as for any call).  FGF_GRAPHS=0 in the environment turns this off.
 */
#ifndef FGF_H
#define FGF_H

#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Status codes (error taxonomy of S:52). */
enum {
    FGF_OK = 0,
    FGF_ERR_PARAM = 1,       /* r < 1, eps not finite or <= 0, s < 1, bad sub_mode,
                                s > 1 and s >= min(H, W) (R7)                       */
    FGF_ERR_SHAPE = 2,       /* batch/H/W < 1, C_I not in {1,3}, C_p not in [1,4]          */
    FGF_ERR_NULL = 3,        /* a required pointer is NULL                                 */
    FGF_ERR_ALIAS = 4,       /* q overlaps I or p (I == p is allowed: self-guidance)       */
    FGF_ERR_ALIGN = 5,       /* a float pointer is not 4-byte aligned                      */
    FGF_ERR_CUDA = 6,        /* a CUDA call or kernel launch failed                        */
    FGF_ERR_NOMEM = 7,       /* workspace too small / device allocation failed             */
    FGF_ERR_NCCL = 8,        /* band path: NCCL missing, or a send/recv/group call failed   */
    FGF_ERR_UNSUPPORTED = 9, /* no engine serves the geometry (colour: r' > 240 with w > 512) */
    FGF_ERR_DEVICE = 10      /* a pointer is not device memory (device entry points) or is
                                not host memory (fgf_filter_host)                           */
};

/* Element type of I, p and q (fgf_filter_ex_ws); every operation is fp32 / fp64. */
enum {
    FGF_F32 = 0,          /* float                                                          */
    FGF_F16 = 1,          /* IEEE binary16 (__half)                                          */
    FGF_BF16 = 2,         /* bfloat16 (__nv_bfloat16)                                        */
    FGF_U8 = 3            /* 8-bit codes: code k is the value fl(k x fl(1/255)); q is
                             stored as the nearest code to 255 q, saturated to [0, 255]
                             (R19; the paper's data are 8-bit images)            */
};

enum {
    FGF_SUB_NEAREST = 0,  /* R3: top-left sample of each s x s block          */
    FGF_SUB_BILINEAR = 1  /* R4: mean of the clipped s x s block              */
};

/* The whole Fast Guided Filter on DEVICE buffers, legacy default stream, internal cached
 * workspace.  I: [batch][C_I][H][W], p: [batch][C_p][H][W], q: [batch][C_p][H][W].
 * r: full-resolution window radius (>= 1); eps: regularisation (> 0, finite, in the
 * squared units of [0,1] intensities); s: subsampling ratio (>= 1; s = 1 is Alg. 1);
 * sub_mode: FGF_SUB_*.  Returns FGF_OK or an FGF_ERR_* code. */
int fgf_filter(const float* I, const float* p, float* q, int batch, int H, int W, int C_I,
               int C_p, int r, double eps, int s, int sub_mode);

/* Bytes of device workspace fgf_filter_ws needs for these arguments (0 on invalid args), the
 * larger of the two subsampling modes.  It takes r, beyond SURVEY §8(b)'s six arguments,
 * because the engine and so the workspace depend on r' (K5's hb rings grow with r'; K5 at
 * s = 1 and K6 need no per-image maps at all). */
size_t fgf_workspace_bytes(int batch, int H, int W, int C_I, int C_p, int r, int s);

/* As fgf_filter, with caller-owned DEVICE workspace (>= fgf_workspace_bytes, 256-byte
 * aligned) and a cudaStream_t passed as void* (NULL = legacy default stream). */
int fgf_filter_ws(const float* I, const float* p, float* q, int batch, int H, int W, int C_I,
                  int C_p, int r, double eps, int s, int sub_mode, void* workspace,
                  size_t ws_bytes, void* cuda_stream);

/* As fgf_filter on HOST buffers (pinned memory gives overlapped transfers; pageable works
 * but serialises).  Streams each image through the device: host->device copy of I, p,
 * the filter, device->host copy of q, overlapped across images on separate streams.
 * Synchronous.  device: CUDA device ordinal to run on.
 * With FGF_SUB_NEAREST and s > 1 the method reads p only at its sample sites p[y s][x s]
 * (the output step P:84-86 uses I alone at full resolution), so only rows y s of p are
 * copied to the device (rows of >= 2 KB; the other rows of the host buffer are not read).
 * One gray frame (batch 1, any element type) with nearest samples is pipelined by rows: the sample rows
 * first, the low-res chain on them while the other rows of I arrive in 8 bands, each band's
 * output rows computed and copied back as soon as its rows are on the device.
 * fgf_filter_host_ex: the same on host buffers of element type dtype (FGF_F32 / FGF_F16 /
 * FGF_BF16 / FGF_U8, the channel combinations of fgf_filter_ex_ws): camera frames stay 8-bit
 * across the host link, 1 + 1/s + 1 bytes per pixel instead of 9 (gray, nearest samples).
 * fgf_filter_host_input_bytes: the host->device bytes one such call copies (0 on invalid
 * arguments; self_guided != 0: p is the same buffer as I). */
int fgf_filter_host(const float* I, const float* p, float* q, int batch, int H, int W, int C_I,
                    int C_p, int r, double eps, int s, int sub_mode, int device);
int fgf_filter_host_ex(const void* I, const void* p, void* q, int batch, int H, int W, int C_I,
                       int C_p, int r, double eps, int s, int sub_mode, int dtype, int device);
size_t fgf_filter_host_input_bytes(int batch, int H, int W, int C_I, int C_p, int r, int s,
                                   int sub_mode, int dtype, int self_guided);

/* Stages 1-5 only: writes the low-res mean maps mean_ab (DEVICE)
 * [batch][C_p][C_I+1][h][w] fp32 -- for p channel c, components j < C_I are mean_a_{c,j}
 * and j = C_I is mean_b_c.  Same validation and workspace rules as fgf_filter_ws. */
int fgf_coefficients(const float* I, const float* p, float* mean_ab, int batch, int H, int W,
                     int C_I, int C_p, int r, double eps, int s, int sub_mode, void* workspace,
                     size_t ws_bytes, void* cuda_stream);

/* Stages 6-7 only: q = upsample(mean_a)^T I + upsample(mean_b) from given DEVICE
 * low-res mean maps laid out as fgf_coefficients writes them (h = ceil(H/s), w = ceil(W/s)).
 * Needs no workspace. */
int fgf_upsample_output(const float* I, const float* mean_ab, float* q, int batch, int H,
                        int W, int C_I, int C_p, int s, void* cuda_stream);

/* ---- Stage entry points for the row-band (multi-GPU, single huge image) path ----
 * A rank that owns full-resolution rows [Y0, Y0 + rows) of an H_total x W image subsamples
 * them (fgf_subsample), exchanges 2r'+1 low-res halo rows of I', p' with its neighbours,
 * runs fgf_lowres_mean on the extended low-res band, and finishes its own rows with
 * fgf_upsample_output_rows, which applies the GLOBAL vertical map of R5. */

/* Step 1 (R3/R4) on `planes` DEVICE planes of H x W -> ceil(H/s) x ceil(W/s).
 * s = 1 copies.  Band rows must start on a multiple of s for the grid to be global. */
int fgf_subsample(const float* src, float* dst, int planes, int H, int W, int s, int sub_mode,
                  void* cuda_stream);

/* Workspace bytes for fgf_lowres_mean. */
size_t fgf_lowres_workspace_bytes(int batch, int h, int w, int C_I, int C_p);

/* Steps 2-5 on given DEVICE low-res planes Is [batch][C_I][h][w] and
 * ps [batch][C_p][h][w] with low-res radius r_low (= r'); writes mean_ab
 * [batch][C_p][C_I+1][h][w].  Windows are clipped at the buffer's own bounds. */
int fgf_lowres_mean(const float* Is, const float* ps, float* mean_ab, int batch, int h, int w,
                    int C_I, int C_p, int r_low, double eps, void* workspace, size_t ws_bytes,
                    void* cuda_stream);

/* Steps 6-7 for full-resolution rows [Y0, Y0 + rows) of an image of height H_total
 * (I, q: DEVICE [batch][C][rows][W]) whose low-res height is h_total and width w, from a maps
 * buffer holding global low-res rows [y0_maps, y0_maps + h_maps) (DEVICE
 * [batch][C_p][C_I+1][h_maps][w]).  FGF_ERR_PARAM if the rows need low-res rows outside it. */
int fgf_upsample_output_rows(const float* I, const float* mean_ab, float* q, int batch, int rows,
                             int W, int C_I, int C_p, int H_total, int h_total, int w, int Y0,
                             int y0_maps, int h_maps, void* cuda_stream);

/* Row-band geometry of rank `rank` of `nranks` for one H x W image (the same
 * rule fgf_filter_band and fgf_filter_bands_loopback use): rank k owns low-res rows
 * [k h / n, (k + 1) h / n) of h = ceil(H/s) (R6) and so full-resolution rows on multiples of s.
 * Host only (no GPU, no launch).  out[10] = {h, w, r', halo = 2r' + 1 + x, own low-res rows y0,
 * y1, own full-res rows Y0, Y1, extended low-res rows e0, e1 of the single exchange}; x = 1 when
 * h s != H (the map scale h / H then exceeds 1 / s and a band's last rows upsample from up to
 * low-res row y1 + 1), else 0.  FGF_ERR_PARAM when a band of several holds fewer than halo
 * low-res rows. */
int fgf_band_geometry(int H, int W, int r, int s, int nranks, int rank, int* out);

/* ---------------------------------------------------------------------------------------
 * One image split into row bands across ranks (BASELINE.json config 4b).
 * Rank `rank` of `nranks` owns full-resolution rows [row0, row0 + rows) of an image of
 * H_total x W (row0 a multiple of s; rows a multiple of s unless the band ends at H_total);
 * with more than one rank every band must span at least halo = 2r'+1+x low-res rows
 * (fgf_band_geometry).  I_band: DEVICE
 * [C_I][rows][W], p_band: [C_p][rows][W] (may equal I_band when C_I = C_p = 1), q_band:
 * [C_p][rows][W], all holding exactly the band's rows.  The call subsamples its rows, sends
 * halo low-res rows of I', p' to rank-1 / rank+1 and receives theirs (ncclSend / ncclRecv in
 * one group on nccl_comm, enqueued on cuda_stream; one exchange, the single-step variant of
 * DESIGN.md §7), runs the low-res chain on the extended band with global window clipping
 * (R1) and writes q for its own rows with the global upsampling map (R5): the result equals
 * the whole-image filter's rows.  nccl_comm is an ncclComm_t (fgf_nccl_comm_init); it may be
 * NULL when nranks = 1.  Workspace: fgf_band_workspace_bytes(), caller-owned device memory.
 * Errors: FGF_ERR_PARAM (band geometry, rank), FGF_ERR_SHAPE, FGF_ERR_NULL, FGF_ERR_ALIGN,
 * FGF_ERR_ALIAS, FGF_ERR_DEVICE, FGF_ERR_NOMEM, FGF_ERR_NCCL (NCCL missing or a call failed),
 * FGF_ERR_CUDA.  The NCCL library is loaded at run time (dlopen "libnccl.so.2"). */
size_t fgf_band_workspace_bytes(int H_total, int W, int row0, int rows, int C_I, int C_p, int r,
                                int s, int nranks);
/* Halo exchange modes of the band path. */
enum {
    FGF_BAND_SINGLE = 0,   /* one exchange: 2r'+1+x rows of I', p' (the default of fgf_filter_band) */
    FGF_BAND_TWO_STEP = 1  /* r' rows of I', p', then ceil(r/s)+1 = r'+1 (+x) rows of a, b
                              (BASELINE.json's halo); the statistics of the halo rows are not
                              recomputed */
};
/* fgf_filter_band with an explicit exchange mode (FGF_ERR_PARAM for an unknown mode).  Every
 * rank must use the same mode; the workspace query covers both. */
int fgf_filter_band_ex(const float* I_band, const float* p_band, float* q_band, int H_total,
                       int W, int row0, int rows, int C_I, int C_p, int r, double eps, int s,
                       int sub_mode, int mode, void* nccl_comm, int rank, int nranks,
                       void* workspace, size_t ws_bytes, void* cuda_stream);
int fgf_filter_band(const float* I_band, const float* p_band, float* q_band, int H_total, int W,
                    int row0, int rows, int C_I, int C_p, int r, double eps, int s, int sub_mode,
                    void* nccl_comm, int rank, int nranks, void* workspace, size_t ws_bytes,
                    void* cuda_stream);
/* NCCL bootstrap for fgf_filter_band: rank 0 creates a 128-byte unique id, the caller
 * distributes it (e.g. torch.distributed broadcast), every rank creates its communicator on
 * its current device.  Return FGF_OK, FGF_ERR_NULL, FGF_ERR_PARAM or FGF_ERR_NCCL. */
int fgf_nccl_unique_id(void* id_out);
int fgf_nccl_comm_init(void** comm_out, const void* id, int rank, int nranks);
int fgf_nccl_comm_destroy(void* comm);
/* Failure detection for the band path: polls ncclCommGetAsyncError on a communicator (the
 * exchange is asynchronous, so a failed peer shows up here, not in fgf_filter_band's status).
 * FGF_OK while healthy or in progress, FGF_ERR_NCCL on an asynchronous NCCL error. */
int fgf_nccl_check(void* comm);
/* Test driver of the band path on ONE device: the nranks bands of a whole image [C][H][W]
 * (batch 1) are filtered one after another with the halo rows copied between the bands'
 * buffers (the same halo geometry fgf_filter_band sends over NCCL), and stitched into q.
 * Band k owns low-res rows [k h / nranks, (k+1) h / nranks).  Workspace:
 * fgf_bands_loopback_workspace_bytes(); mode as fgf_filter_band_ex. */
size_t fgf_bands_loopback_workspace_bytes(int H, int W, int C_I, int C_p, int r, int s,
                                          int nranks);
int fgf_filter_bands_loopback(const float* I, const float* p, float* q, int H, int W, int C_I,
                              int C_p, int r, double eps, int s, int sub_mode, int mode,
                              int nranks, void* workspace, size_t ws_bytes, void* cuda_stream);

/* Reduced-precision I/O: fgf_filter_ws with I, p and q of element type
 * dtype (FGF_F32 / FGF_F16 / FGF_BF16 / FGF_U8; all three buffers the same type, aligned to
 * the element size).  Only the storage changes: samples are widened to fp32 / fp64 on load
 * exactly as in the fp32 path (8-bit code k -> fl(k x fl(1/255))), and q is rounded to the element type
 * once, on store (8-bit: nearest code, saturated).  The reduced types support C_I / C_p =
 * 1 / 1, 3 / 1 and 3 / 3 (else FGF_ERR_UNSUPPORTED).  Workspace: fgf_workspace_bytes_ex().
 * Other errors as fgf_filter_ws; a bad dtype is FGF_ERR_PARAM. */
size_t fgf_workspace_bytes_ex(int batch, int H, int W, int C_I, int C_p, int r, int s, int dtype);
int fgf_filter_ex_ws(const void* I, const void* p, void* q, int batch, int H, int W, int C_I,
                     int C_p, int r, double eps, int s, int sub_mode, int dtype, void* workspace,
                     size_t ws_bytes, void* cuda_stream);

/* Joint upsampling (the setting P:18 names as the origin of the speed-up,
 * procedure not given in the paper -- DESIGN.md R18): the filtering input is given ONLY at
 * low resolution, p_low: DEVICE [batch][C_p][h][w] with h = ceil(H/s), w = ceil(W/s), and is
 * taken as the p' of Alg. 2; I' = f_sub(I, s) (sub_mode), steps 2-5 on (I', p'), steps 6-7
 * with the full-resolution I: q [batch][C_p][H][W].  Workspace: fgf_joint_workspace_bytes().
 * Errors as fgf_filter_ws. */
size_t fgf_joint_workspace_bytes(int batch, int H, int W, int C_I, int C_p, int r, int s);
int fgf_filter_joint_ws(const float* I, const float* p_low, float* q, int batch, int H, int W,
                        int C_I, int C_p, int r, double eps, int s, int sub_mode,
                        void* workspace, size_t ws_bytes, void* cuda_stream);

/* Detail enhancement, the application of PAPER.md Fig. 2 ("enhanced images with x5
 * detail"; SPEC S:303-311 enhance): out = (I - q) * gain + q, with q the SELF-guided fast
 * guided filter of I (p = I, C_p = C_I = C in {1, 3}) with these r, eps, s, sub_mode.  Since
 * out = gain I + (1 - gain)(mean_a^T I + mean_b), the enhancement is folded into the mean
 * maps as they are written (a_cc -> (1 - gain) a_cc + gain, the rest scaled by 1 - gain):
 * same kernels, same HBM bytes as fgf_filter_ws.  gain = 1 returns I exactly, gain = 0 is
 * the filter.  DEVICE buffers I, out: [batch][C][H][W]; out may not overlap I; no clamp
 * (S:266).  Workspace as fgf_filter_ws (fgf_workspace_bytes(batch, H, W, C, C, r, s)).
 * Errors: as fgf_filter_ws; gain < 0 or not finite -> FGF_ERR_PARAM. */
int fgf_enhance_ws(const float* I, float* out, int batch, int H, int W, int C, int r,
                   double eps, int s, int sub_mode, double gain, void* workspace,
                   size_t ws_bytes, void* cuda_stream);

/* Guidance of detail enhancement: the image itself (colour guidance for RGB, R20),
 * or SPEC's shared gray guidance to_grayscale(img) = 0.299 R + 0.587 G + 0.114 B (S:48-51,
 * S:297) with the three channels as the filtering input. */
enum { FGF_GUIDE_SELF = 0, FGF_GUIDE_LUMA = 1 };

/* fgf_enhance_ws with a choice of guidance.  FGF_GUIDE_SELF (or C = 1) is fgf_enhance_ws.
 * FGF_GUIDE_LUMA with C = 3: a luminance kernel writes L into the workspace, the filter runs
 * with I = L (C_I = 1) and p = the image (C_p = 3), and a blend kernel forms
 * out = gain img + (1 - gain) q in place (three kernels' worth of extra traffic: the gain does
 * not fold into the maps when the guidance is not the image).  Workspace:
 * fgf_enhance_workspace_bytes (0 on invalid args).  Errors as fgf_enhance_ws; a bad guide is
 * FGF_ERR_PARAM. */
size_t fgf_enhance_workspace_bytes(int batch, int H, int W, int C, int r, int s, int guide);
int fgf_enhance_ex_ws(const float* I, float* out, int batch, int H, int W, int C, int r,
                      double eps, int s, int sub_mode, double gain, int guide, void* workspace,
                      size_t ws_bytes, void* cuda_stream);

/* Diagnostics (single-threaded use): per-kernel CUDA-event timing of the launches this
 * process enqueues.  fgf_profile_enable(1) clears old records and starts recording an event
 * pair around every kernel launch on its launching stream; fgf_profile_enable(0) stops.
 * fgf_profile_read() waits for the recorded events and writes, for each kernel kind
 * (0 = subsample K0 (and the luminance kernel), 1 = statistics + coefficients K1, 2 = box of
 * a, b K3, 3 = upsample + output K4 (and the enhance blend), 4 = fused low-res chain K13 for
 * gray guidance, 5 = K5, 6 = K6), the summed device milliseconds and the launch count, then
 * clears the records.  Returns the number of kinds written (<= max_kinds) or -FGF_ERR_CUDA. */
int fgf_profile_enable(int on);
int fgf_profile_read(double* ms, int* launches, int max_kinds);

/* Number of kernel launches the last successful call on this thread enqueued. */
int fgf_last_launch_count(void);

/* Static description of a status code. */
const char* fgf_status_str(int status);

/* Library version string. */
const char* fgf_version(void);

#ifdef __cplusplus
}
#endif

#endif /* FGF_H */
