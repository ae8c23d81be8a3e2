/*
 * fgf_oracle.c -- plain, slow, obviously-correct double-precision CPU oracle of
 * the Fast Guided Filter (K. He, J. Sun, "Fast Guided Filter", arXiv 1505.00996).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library.  The product path
 * (paper_1505_00996_b200/, libfgf.so) never links, imports or calls it, and this
 * file shares no code, header, table or helper with the CUDA path.
 *
 * Citation keys: P:n = PAPER.md line n (LaTeX source of the note),
 *                S:n = SPEC.md line n, DESIGN.md Rn = reading n in DESIGN.md.
 *
 * What it computes (Alg. 2, with I = guidance, p = input, q = output):
 *   1  I' = f_subsample(I, s), p' = f_subsample(p, s), r' = r/s
 *   2  mean_I = f_mean(I', r'), mean_p = f_mean(p', r'),
 *      corr_I = f_mean(I'.*I', r'), corr_Ip = f_mean(I'.*p', r')
 *   3  var_I = corr_I - mean_I.*mean_I, cov_Ip = corr_Ip - mean_I.*mean_p
 *   4  a = cov_Ip ./ (var_I + eps), b = mean_p - a.*mean_I             (Eq.2-3)
 *   5  mean_a = f_mean(a, r'), mean_b = f_mean(b, r')
 *   6  mean_a, mean_b = f_upsample(., s)  (bilinear)
 *   7  q = mean_a .* I + mean_b with the FULL-resolution I
 * Color guidance (C_I = 3) replaces 3-4 by the ridge-regression solve of the cited
 * journal version [He2013] (cited at P:41, not in the container): DESIGN.md R9.
 *
 * Readings where the paper is silent (all listed in DESIGN.md "Readings"):
 *   R1 box border: clip-and-renormalize, divide by the in-bounds count
 *   R2 r' = max(1, floor(r/s + 1/2))
 *   R3 nearest subsample takes the top-left sample I[y*s][x*s]
 *   R4 "bilinear" subsample = mean of the clipped s x s block
 *   R5 upsample map x_src = (x + 1/2) * w/W - 1/2 clamped to [0, w-1]
 *   R6 low-res dims ceil(H/s) x ceil(W/s)
 *   R8 gray: clamp var_I < 0 to 0 (only var, not cov)
 *   R9 color: a = (Sigma + eps U)^-1 (corr_Ip - mu p_bar), b = p_bar - a^T mu, solved by
 *      Gaussian elimination with partial pivoting (NOT the adjugate the GPU uses)
 *   R10 several p channels: independent a_c, b_c per p channel
 *   R11 no output clamp
 *
 * Precision: IEEE double, compiled with -O2 -ffp-contract=off and no fast-math.
 * Parallelism: OpenMP over rows / planes only; every output value is computed by
 * the same sequence of operations regardless of the thread count.
 *
 * All image arrays are planar, row-major: [batch][C][H][W].
 */
#include <math.h>
#include <stdlib.h>
#include <string.h>

#define FGFO_OK 0
#define FGFO_EINVAL (-1)
#define FGFO_ENOMEM (-2)

/* R6: low-resolution size. */
int fgfo_lowres_dim(int D, int s) { return (D + s - 1) / s; }

/* R2 ("r' = r/s"): round half up, floor of 1.
 * floor(r/s + 1/2) == floor((2r + s) / (2s)) for positive integers. */
int fgfo_radius_lowres(int r, int s) {
    int rr = (2 * r + s) / (2 * s);
    return rr < 1 ? 1 : rr;
}

/* Step 1, one plane.  mode 0 = nearest (R3), 1 = block mean (R4). */
void fgfo_subsample(const double* src, int H, int W, int s, int mode, double* dst) {
    int h = fgfo_lowres_dim(H, s), w = fgfo_lowres_dim(W, s);
    for (int y = 0; y < h; ++y) {
        for (int x = 0; x < w; ++x) {
            if (mode == 0) {
                dst[(size_t)y * w + x] = src[(size_t)(y * s) * W + (size_t)(x * s)];
            } else {
                int y1 = y * s + s < H ? y * s + s : H;
                int x1 = x * s + s < W ? x * s + s : W;
                double sum = 0.0;
                int count = 0;
                for (int yy = y * s; yy < y1; ++yy)
                    for (int xx = x * s; xx < x1; ++xx) {
                        sum += src[(size_t)yy * W + xx];
                        ++count;
                    }
                dst[(size_t)y * w + x] = sum / (double)count;
            }
        }
    }
}

/* f_mean(X, r) ("a mean filter with a radius r"; R1 clip-and-renormalize):
 *   out[y][x] = (1/|Omega|) sum_{(u,v) in Omega} X[u][v],
 *   Omega = ([y-r, y+r] ∩ [0,h)) x ([x-r, x+r] ∩ [0,w)).
 * O(hw) with prefix sums: first along each row, then down each column of the
 * row-window sums ("O(N) ... independent of the filter size"). */
int fgfo_box_mean(const double* X, int h, int w, int r, double* out) {
    double* rowsum = (double*)malloc(sizeof(double) * (size_t)h * w);
    if (!rowsum) return FGFO_ENOMEM;
    #pragma omp parallel
    {
        double* pre = (double*)malloc(sizeof(double) * (size_t)((h > w ? h : w) + 1));
        #pragma omp for
        for (int y = 0; y < h; ++y) {
            pre[0] = 0.0;
            for (int x = 0; x < w; ++x) pre[x + 1] = pre[x] + X[(size_t)y * w + x];
            for (int x = 0; x < w; ++x) {
                int x0 = x - r < 0 ? 0 : x - r;
                int x1 = x + r > w - 1 ? w - 1 : x + r;
                rowsum[(size_t)y * w + x] = pre[x1 + 1] - pre[x0];
            }
        }
        #pragma omp for
        for (int x = 0; x < w; ++x) {
            pre[0] = 0.0;
            for (int y = 0; y < h; ++y) pre[y + 1] = pre[y] + rowsum[(size_t)y * w + x];
            int x0 = x - r < 0 ? 0 : x - r;
            int x1 = x + r > w - 1 ? w - 1 : x + r;
            for (int y = 0; y < h; ++y) {
                int y0 = y - r < 0 ? 0 : y - r;
                int y1 = y + r > h - 1 ? h - 1 : y + r;
                double count = (double)(y1 - y0 + 1) * (double)(x1 - x0 + 1);
                out[(size_t)y * w + x] = (pre[y1 + 1] - pre[y0]) / count;
            }
        }
        free(pre);
    }
    free(rowsum);
    return FGFO_OK;
}

/* R5: source coordinate of destination index d for a resize
 * of n_src -> n_dst samples, pixel-centre aligned, clamped. */
static void upsample_coord(int d, int n_src, int n_dst, int* i0, int* i1, double* f) {
    double c = ((double)d + 0.5) * (double)n_src / (double)n_dst - 0.5;
    if (c < 0.0) c = 0.0;
    if (c > (double)(n_src - 1)) c = (double)(n_src - 1);
    int lo = (int)floor(c);
    *i0 = lo;
    *i1 = lo + 1 < n_src ? lo + 1 : n_src - 1;
    *f = c - (double)lo;
}

/* Step 6 ("bilinearly upsampled to the original size"), one plane. */
void fgfo_upsample(const double* src, int h, int w, int H, int W, double* dst) {
    #pragma omp parallel for
    for (int Y = 0; Y < H; ++Y) {
        int y0, y1;
        double fy;
        upsample_coord(Y, h, H, &y0, &y1, &fy);
        for (int X = 0; X < W; ++X) {
            int x0, x1;
            double fx;
            upsample_coord(X, w, W, &x0, &x1, &fx);
            dst[(size_t)Y * W + X] =
                (1.0 - fy) * (1.0 - fx) * src[(size_t)y0 * w + x0] +
                (1.0 - fy) * fx * src[(size_t)y0 * w + x1] +
                fy * (1.0 - fx) * src[(size_t)y1 * w + x0] +
                fy * fx * src[(size_t)y1 * w + x1];
        }
    }
}

/* R9: solve (M) a = v for one 3x3 system by Gaussian elimination with partial
 * pivoting.  M is overwritten. */
static void solve3(double M[3][3], double v[3], double a[3]) {
    for (int k = 0; k < 3; ++k) {
        int piv = k;
        for (int i = k + 1; i < 3; ++i)
            if (fabs(M[i][k]) > fabs(M[piv][k])) piv = i;
        if (piv != k) {
            for (int j = 0; j < 3; ++j) {
                double t = M[k][j]; M[k][j] = M[piv][j]; M[piv][j] = t;
            }
            double t = v[k]; v[k] = v[piv]; v[piv] = t;
        }
        for (int i = k + 1; i < 3; ++i) {
            double m = M[i][k] / M[k][k];
            for (int j = k; j < 3; ++j) M[i][j] -= m * M[k][j];
            v[i] -= m * v[k];
        }
    }
    for (int i = 2; i >= 0; --i) {
        double acc = v[i];
        for (int j = i + 1; j < 3; ++j) acc -= M[i][j] * a[j];
        a[i] = acc / M[i][i];
    }
}

static int check_args(int batch, int H, int W, int C_I, int C_p, int r, double eps, int s,
                      int sub_mode) {
    if (batch < 1 || H < 1 || W < 1) return FGFO_EINVAL;
    if (C_I != 1 && C_I != 3) return FGFO_EINVAL;
    if (C_p < 1 || C_p > 4) return FGFO_EINVAL;
    if (r < 1 || !(eps > 0.0) || s < 1 || (sub_mode != 0 && sub_mode != 1)) return FGFO_EINVAL;
    if (s > 1 && (s >= H || s >= W)) return FGFO_EINVAL; /* S:246, R7 */
    return FGFO_OK;
}

/* Steps 2-5 of Alg. 2 for one image, on given fp64 low-res planes
 * Is: [C_I][h][w] (I') and ps: [C_p][h][w] (p'), radius rl = r'.  Outputs low-res maps
 * [C_p][C_I+1][h][w]: for each p channel c the C_I components of a_c (mean_a_c) followed
 * by b_c (mean_b_c).  ab may be NULL. */
static int lowres_chain_one(const double* Is, const double* ps, int h, int w, int C_I,
                            int C_p, int rl, double eps, double* ab, double* mean_ab) {
    const size_t n = (size_t)h * w;
    int rc = FGFO_OK;

    double* tmp = (double*)malloc(sizeof(double) * n);
    double* meanI = (double*)malloc(sizeof(double) * n * C_I);
    double* corrII = (double*)malloc(sizeof(double) * n * C_I * C_I);
    double* meanp = (double*)malloc(sizeof(double) * n);
    double* corrIp = (double*)malloc(sizeof(double) * n * C_I);
    double* coef = (double*)malloc(sizeof(double) * n * (C_I + 1));
    if (!tmp || !meanI || !corrII || !meanp || !corrIp || !coef) {
        rc = FGFO_ENOMEM;
        goto done;
    }

    /* Step 2 (guidance part): mean_I = f(I'), corr_I = f(I'.*I') (all j,k pairs). */
    for (int j = 0; j < C_I; ++j) {
        if ((rc = fgfo_box_mean(Is + (size_t)j * n, h, w, rl, meanI + (size_t)j * n))) goto done;
        for (int k = 0; k < C_I; ++k) {
            for (size_t i = 0; i < n; ++i) tmp[i] = Is[(size_t)j * n + i] * Is[(size_t)k * n + i];
            if ((rc = fgfo_box_mean(tmp, h, w, rl, corrII + ((size_t)j * C_I + k) * n))) goto done;
        }
    }

    for (int c = 0; c < C_p; ++c) {
        const double* pc = ps + (size_t)c * n;
        /* Step 2 (input part): mean_p = f(p'), corr_Ip = f(I'.*p'). */
        if ((rc = fgfo_box_mean(pc, h, w, rl, meanp))) goto done;
        for (int j = 0; j < C_I; ++j) {
            for (size_t i = 0; i < n; ++i) tmp[i] = Is[(size_t)j * n + i] * pc[i];
            if ((rc = fgfo_box_mean(tmp, h, w, rl, corrIp + (size_t)j * n))) goto done;
        }
        /* Steps 3-4. */
        for (size_t i = 0; i < n; ++i) {
            if (C_I == 1) {
                double var = corrII[i] - meanI[i] * meanI[i];      /* var_I */
                if (var < 0.0) var = 0.0;                           /* R8 */
                double cov = corrIp[i] - meanI[i] * meanp[i];       /* cov_Ip */
                double a = cov / (var + eps);                        /* Eq.2 */
                coef[i] = a;
                coef[n + i] = meanp[i] - a * meanI[i];               /* Eq.3 */
            } else {
                double M[3][3], v[3], a[3];
                for (int j = 0; j < 3; ++j) {
                    for (int k = 0; k < 3; ++k)
                        M[j][k] = corrII[((size_t)j * 3 + k) * n + i] -
                                  meanI[(size_t)j * n + i] * meanI[(size_t)k * n + i];
                    M[j][j] += eps;                                  /* Sigma + eps U */
                    v[j] = corrIp[(size_t)j * n + i] - meanI[(size_t)j * n + i] * meanp[i];
                }
                solve3(M, v, a);
                double b = meanp[i];
                for (int j = 0; j < 3; ++j) {
                    coef[(size_t)j * n + i] = a[j];
                    b -= a[j] * meanI[(size_t)j * n + i];
                }
                coef[(size_t)3 * n + i] = b;
            }
        }
        /* Step 5: mean_a = f(a), mean_b = f(b). */
        for (int m = 0; m <= C_I; ++m) {
            double* dst = mean_ab + ((size_t)c * (C_I + 1) + m) * n;
            if (ab) memcpy(ab + ((size_t)c * (C_I + 1) + m) * n, coef + (size_t)m * n, sizeof(double) * n);
            if ((rc = fgfo_box_mean(coef + (size_t)m * n, h, w, rl, dst))) goto done;
        }
    }
done:
    free(tmp); free(meanI); free(corrII); free(meanp); free(corrIp); free(coef);
    return rc;
}

/* Steps 1-5 of Alg. 2 for one image.  Ip: [C_I][H][W], pp: [C_p][H][W] (float, widened
 * to double).  Step 1 into fp64 planes, then steps 2-5 (lowres_chain_one). */
static int coefficients_one(const float* Ip, const float* pp, int H, int W, int C_I, int C_p,
                            int r, double eps, int s, int sub_mode, double* ab,
                            double* mean_ab) {
    const int h = fgfo_lowres_dim(H, s), w = fgfo_lowres_dim(W, s);
    const size_t N = (size_t)H * W, n = (size_t)h * w;
    int rc = FGFO_ENOMEM;
    double* full = (double*)malloc(sizeof(double) * N);
    double* Is = (double*)malloc(sizeof(double) * n * C_I);   /* I' */
    double* ps = (double*)malloc(sizeof(double) * n * C_p);   /* p' */
    if (full && Is && ps) {
        /* Step 1: I' = f_subsample(I, s), p' = f_subsample(p, s). */
        for (int j = 0; j < C_I; ++j) {
            for (size_t i = 0; i < N; ++i) full[i] = (double)Ip[(size_t)j * N + i];
            fgfo_subsample(full, H, W, s, sub_mode, Is + (size_t)j * n);
        }
        for (int c = 0; c < C_p; ++c) {
            for (size_t i = 0; i < N; ++i) full[i] = (double)pp[(size_t)c * N + i];
            fgfo_subsample(full, H, W, s, sub_mode, ps + (size_t)c * n);
        }
        rc = lowres_chain_one(Is, ps, h, w, C_I, C_p, fgfo_radius_lowres(r, s), eps, ab, mean_ab);
    }
    free(full); free(Is); free(ps);
    return rc;
}

/* Steps 2-5 of Alg. 2 over a batch of given fp64 low-res planes
 * Is [batch][C_I][h][w], ps [batch][C_p][h][w] with radius rl: the low-res chain of joint
 * upsampling (R18), where p' is an input and I' = f_sub(I, s) stays in double. */
int fgfo_lowres_chain(const double* Is, const double* ps, int batch, int h, int w, int C_I,
                      int C_p, int rl, double eps, double* mean_ab) {
    if (batch < 1 || h < 1 || w < 1 || (C_I != 1 && C_I != 3) || C_p < 1 || C_p > 4 || rl < 1 ||
        !(eps > 0.0))
        return FGFO_EINVAL;
    const size_t n = (size_t)h * w, per = n * (size_t)C_p * (C_I + 1);
    for (int b = 0; b < batch; ++b) {
        int rc = lowres_chain_one(Is + (size_t)b * C_I * n, ps + (size_t)b * C_p * n, h, w, C_I,
                                  C_p, rl, eps, NULL, mean_ab + b * per);
        if (rc) return rc;
    }
    return FGFO_OK;
}

/* Steps 6-7 for one image: upsample every low-res mean map, then
 * q_c = sum_j mean_a_{c,j} .* I_j + mean_b_c  with the full-resolution I. */
static int output_one(const float* Ip, const double* mean_ab, int H, int W, int h, int w,
                      int C_I, int C_p, double* q) {
    const size_t N = (size_t)H * W, n = (size_t)h * w;
    double* up = (double*)malloc(sizeof(double) * N);
    if (!up) return FGFO_ENOMEM;
    for (int c = 0; c < C_p; ++c) {
        double* qc = q + (size_t)c * N;
        /* mean_b_c */
        fgfo_upsample(mean_ab + ((size_t)c * (C_I + 1) + C_I) * n, h, w, H, W, up);
        for (size_t i = 0; i < N; ++i) qc[i] = up[i];
        for (int j = 0; j < C_I; ++j) {
            fgfo_upsample(mean_ab + ((size_t)c * (C_I + 1) + j) * n, h, w, H, W, up);
            for (size_t i = 0; i < N; ++i) qc[i] = up[i] * (double)Ip[(size_t)j * N + i] + qc[i];
        }
    }
    free(up);
    return FGFO_OK;
}

/* Alg. 2 steps 1-5 over a batch: a, b (optional) and mean_a, mean_b low-res maps,
 * each [batch][C_p][C_I+1][h][w] double. */
int fgfo_coefficients(const float* I, const float* p, int batch, int H, int W, int C_I, int C_p,
                      int r, double eps, int s, int sub_mode, double* ab, double* mean_ab) {
    int rc = check_args(batch, H, W, C_I, C_p, r, eps, s, sub_mode);
    if (rc) return rc;
    const size_t N = (size_t)H * W;
    const size_t n = (size_t)fgfo_lowres_dim(H, s) * fgfo_lowres_dim(W, s);
    const size_t per = n * (size_t)C_p * (C_I + 1);
    for (int b = 0; b < batch; ++b) {
        rc = coefficients_one(I + (size_t)b * C_I * N, p + (size_t)b * C_p * N, H, W, C_I, C_p, r,
                              eps, s, sub_mode, ab ? ab + b * per : NULL, mean_ab + b * per);
        if (rc) return rc;
    }
    return FGFO_OK;
}

/* Alg. 2 steps 6-7 over a batch, from given low-res mean maps. */
int fgfo_upsample_output(const float* I, const double* mean_ab, double* q, int batch, int H,
                         int W, int C_I, int C_p, int s) {
    if (batch < 1 || H < 1 || W < 1 || s < 1 || (C_I != 1 && C_I != 3) || C_p < 1 || C_p > 4)
        return FGFO_EINVAL;
    const int h = fgfo_lowres_dim(H, s), w = fgfo_lowres_dim(W, s);
    const size_t N = (size_t)H * W, n = (size_t)h * w;
    for (int b = 0; b < batch; ++b) {
        int rc = output_one(I + (size_t)b * C_I * N, mean_ab + (size_t)b * C_p * (C_I + 1) * n, H,
                            W, h, w, C_I, C_p, q + (size_t)b * C_p * N);
        if (rc) return rc;
    }
    return FGFO_OK;
}

/* The whole Fast Guided Filter (Alg. 2); s = 1 is the guided filter (Alg. 1). */
int fgfo_filter(const float* I, const float* p, double* q, int batch, int H, int W, int C_I,
                int C_p, int r, double eps, int s, int sub_mode) {
    int rc = check_args(batch, H, W, C_I, C_p, r, eps, s, sub_mode);
    if (rc) return rc;
    const int h = fgfo_lowres_dim(H, s), w = fgfo_lowres_dim(W, s);
    const size_t N = (size_t)H * W, n = (size_t)h * w;
    const size_t per = n * (size_t)C_p * (C_I + 1);
    double* mean_ab = (double*)malloc(sizeof(double) * per);
    if (!mean_ab) return FGFO_ENOMEM;
    for (int b = 0; b < batch && !rc; ++b) {
        const float* Ib = I + (size_t)b * C_I * N;
        rc = coefficients_one(Ib, p + (size_t)b * C_p * N, H, W, C_I, C_p, r, eps, s, sub_mode,
                              NULL, mean_ab);
        if (!rc) rc = output_one(Ib, mean_ab, H, W, h, w, C_I, C_p, q + (size_t)b * C_p * N);
    }
    free(mean_ab);
    return rc;
}

/* The whole Fast Guided Filter (Alg. 2) on fp64 inputs: I [batch][C_I][H][W] and
 * p [batch][C_p][H][W] in double (e.g. a guidance computed in double, such as SPEC's
 * to_grayscale luminance).  The same steps as fgfo_filter -- step 1 by
 * fgfo_subsample, steps 2-5 by lowres_chain_one, steps 6-7 by fgfo_upsample and the product
 * with the full-resolution I -- with no rounding of the inputs to fp32. */
int fgfo_filter_f64(const double* I, const double* p, double* q, int batch, int H, int W,
                    int C_I, int C_p, int r, double eps, int s, int sub_mode) {
    int rc = check_args(batch, H, W, C_I, C_p, r, eps, s, sub_mode);
    if (rc) return rc;
    const int h = fgfo_lowres_dim(H, s), w = fgfo_lowres_dim(W, s);
    const size_t N = (size_t)H * W, n = (size_t)h * w;
    double* Is = (double*)malloc(sizeof(double) * n * C_I);
    double* ps = (double*)malloc(sizeof(double) * n * C_p);
    double* mean_ab = (double*)malloc(sizeof(double) * n * C_p * (C_I + 1));
    double* up = (double*)malloc(sizeof(double) * N);
    rc = (Is && ps && mean_ab && up) ? FGFO_OK : FGFO_ENOMEM;
    for (int b = 0; b < batch && !rc; ++b) {
        const double* Ib = I + (size_t)b * C_I * N;
        const double* pb = p + (size_t)b * C_p * N;
        double* qb = q + (size_t)b * C_p * N;
        for (int j = 0; j < C_I; ++j) fgfo_subsample(Ib + (size_t)j * N, H, W, s, sub_mode, Is + (size_t)j * n);
        for (int c = 0; c < C_p; ++c) fgfo_subsample(pb + (size_t)c * N, H, W, s, sub_mode, ps + (size_t)c * n);
        rc = lowres_chain_one(Is, ps, h, w, C_I, C_p, fgfo_radius_lowres(r, s), eps, NULL, mean_ab);
        for (int c = 0; c < C_p && !rc; ++c) {
            double* qc = qb + (size_t)c * N;
            fgfo_upsample(mean_ab + ((size_t)c * (C_I + 1) + C_I) * n, h, w, H, W, up);   /* mean_b */
            for (size_t i = 0; i < N; ++i) qc[i] = up[i];
            for (int j = 0; j < C_I; ++j) {
                fgfo_upsample(mean_ab + ((size_t)c * (C_I + 1) + j) * n, h, w, H, W, up);
                for (size_t i = 0; i < N; ++i) qc[i] = up[i] * Ib[(size_t)j * N + i] + qc[i];
            }
        }
    }
    free(Is); free(ps); free(mean_ab); free(up);
    return rc;
}
