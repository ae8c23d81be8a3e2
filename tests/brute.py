"""Brute-force references used to PIN the oracle (never the CUDA path directly).

They are deliberately a different computation from oracle/fgf_oracle.c:
  * window averages by explicit double loops over pixel lists (no prefix sums);
  * the guided-filter coefficients by solving, per window, the ridge regression the
    paper says Eq.2-3 minimise ("minimizing the reconstruction error"; the
    energy of [He2010]: sum_{i in w_k} (a^T I_i + b - p_i)^2 + eps |a|^2) with
    numpy.linalg.lstsq on the stacked pixel list -- not the closed form of Eq.2;
  * upsampling as separable interpolation matrices U_y M U_x^T.
Only small images (<= ~64x64) are fed to these.
"""
from __future__ import annotations

import numpy as np


def window(y, x, h, w, r):
    """Clipped window rows/cols around (y, x) (R1)."""
    return range(max(0, y - r), min(h, y + r + 1)), range(max(0, x - r), min(w, x + r + 1))


def box_brute(X, r):
    X = np.asarray(X, np.float64)
    h, w = X.shape
    out = np.empty_like(X)
    for y in range(h):
        for x in range(w):
            rows, cols = window(y, x, h, w, r)
            acc = 0.0
            cnt = 0
            for u in rows:
                for v in cols:
                    acc += X[u, v]
                    cnt += 1
            out[y, x] = acc / cnt
    return out


def ridge_coefficients(I, p, r, eps):
    """Per-window ridge regression (Eq.1-3).  I: [C_I,h,w], p: [h,w].
    Returns a: [C_I,h,w], b: [h,w]."""
    I = np.asarray(I, np.float64)
    p = np.asarray(p, np.float64)
    C, h, w = I.shape
    a = np.empty((C, h, w))
    b = np.empty((h, w))
    for y in range(h):
        for x in range(w):
            rows, cols = window(y, x, h, w, r)
            pix = [(u, v) for u in rows for v in cols]
            n = len(pix)
            # rows: [I_i^T, 1] -> p_i ; regulariser rows: sqrt(n*eps) e_j -> 0
            # (eps a^2 inside the sum over the n pixels of the window, [He2010]).
            A = np.zeros((n + C, C + 1))
            t = np.zeros(n + C)
            for k, (u, v) in enumerate(pix):
                A[k, :C] = I[:, u, v]
                A[k, C] = 1.0
                t[k] = p[u, v]
            for j in range(C):
                A[n + j, j] = np.sqrt(n * eps)
            sol = np.linalg.lstsq(A, t, rcond=None)[0]
            a[:, y, x] = sol[:C]
            b[y, x] = sol[C]
    return a, b


def guided_filter_brute(I, p, r, eps):
    """Alg. 1 / Eq.4: q_i = mean over windows containing i of (a_k^T I_i + b_k)."""
    I = np.asarray(I, np.float64)
    if I.ndim == 2:
        I = I[None]
    a, b = ridge_coefficients(I, p, r, eps)
    abar = np.stack([box_brute(a[j], r) for j in range(I.shape[0])])
    bbar = box_brute(b, r)
    return (abar * I).sum(0) + bbar


def lowres_radius(r, s):
    return max(1, (2 * r + s) // (2 * s))


def subsample_brute(X, s, mode):
    X = np.asarray(X, np.float64)
    H, W = X.shape
    if mode == 0:
        return X[::s, ::s].copy()
    h, w = -(-H // s), -(-W // s)
    out = np.empty((h, w))
    for y in range(h):
        for x in range(w):
            out[y, x] = X[y * s:min(H, y * s + s), x * s:min(W, x * s + s)].mean()
    return out


def interp_matrix(n_dst, n_src):
    """1-D pixel-centre bilinear interpolation matrix: row d has weights on
    floor(c) and floor(c)+1 with c = clamp((d+1/2) n_src/n_dst - 1/2, 0, n_src-1)."""
    U = np.zeros((n_dst, n_src))
    for d in range(n_dst):
        c = min(max((d + 0.5) * n_src / n_dst - 0.5, 0.0), n_src - 1.0)
        lo = int(np.floor(c))
        hi = min(lo + 1, n_src - 1)
        f = c - lo
        U[d, lo] += 1.0 - f
        U[d, hi] += f
    return U


def upsample_brute(M, H, W):
    M = np.asarray(M, np.float64)
    h, w = M.shape
    return interp_matrix(H, h) @ M @ interp_matrix(W, w).T


def fast_guided_filter_brute(I, p, r, eps, s, mode=0):
    """Alg. 2 composed from the brute-force pieces above."""
    I = np.asarray(I, np.float64)
    if I.ndim == 2:
        I = I[None]
    C, H, W = I.shape
    rl = lowres_radius(r, s)
    Is = np.stack([subsample_brute(I[j], s, mode) for j in range(C)])
    ps = subsample_brute(p, s, mode)
    a, b = ridge_coefficients(Is, ps, rl, eps)
    abar = np.stack([upsample_brute(box_brute(a[j], rl), H, W) for j in range(C)])
    bbar = upsample_brute(box_brute(b, rl), H, W)
    return (abar * I).sum(0) + bbar
