"""ctypes wrapper of the double-precision CPU oracle (oracle/fgf_oracle.c).

TEST INFRASTRUCTURE ONLY: only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / ``--impl reference`` legs may import this package.  The product
path (paper_1505_00996_b200) never imports it and shares no code with it.

Every function follows Alg. 2 of the paper step by step;
see the header of fgf_oracle.c for the passage each step cites and the
readings (R1-R11) where the paper is silent.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "fgf_oracle.c")
_LIB = os.path.join(_HERE, "libfgf_oracle.so")

NEAREST = 0
BLOCKMEAN = 1  # the SPEC reading of "bilinear" subsampling


def build(force: bool = False) -> str:
    """Compile the oracle with gcc: IEEE double, no FMA contraction, no fast-math."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        cmd = ["gcc", "-O2", "-std=c11", "-ffp-contract=off", "-fno-fast-math", "-fopenmp",
               "-shared", "-fPIC", "-o", _LIB, _SRC, "-lm"]
        subprocess.check_call(cmd)
    return _LIB


_lib = None


def _load():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_LIB)
        D = ctypes.POINTER(ctypes.c_double)
        F = ctypes.POINTER(ctypes.c_float)
        i, d = ctypes.c_int, ctypes.c_double
        lib.fgfo_lowres_dim.argtypes = [i, i]
        lib.fgfo_radius_lowres.argtypes = [i, i]
        lib.fgfo_subsample.argtypes = [D, i, i, i, i, D]
        lib.fgfo_subsample.restype = None
        lib.fgfo_box_mean.argtypes = [D, i, i, i, D]
        lib.fgfo_upsample.argtypes = [D, i, i, i, i, D]
        lib.fgfo_upsample.restype = None
        lib.fgfo_coefficients.argtypes = [F, F, i, i, i, i, i, i, d, i, i, D, D]
        lib.fgfo_upsample_output.argtypes = [F, D, D, i, i, i, i, i, i]
        lib.fgfo_filter.argtypes = [F, F, D, i, i, i, i, i, i, d, i, i]
        lib.fgfo_lowres_chain.argtypes = [D, D, i, i, i, i, i, i, d, D]
        lib.fgfo_filter_f64.argtypes = [D, D, D, i, i, i, i, i, i, d, i, i]
        _lib = lib
    return _lib


def _dptr(a):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def _fptr(a):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_float))


def _f32(a):
    return np.ascontiguousarray(np.asarray(a, dtype=np.float32))


def _f64(a):
    return np.ascontiguousarray(np.asarray(a, dtype=np.float64))


def lowres_dim(D: int, s: int) -> int:
    """R6: ceil(D/s)."""
    return _load().fgfo_lowres_dim(D, s)


def radius_lowres(r: int, s: int) -> int:
    """R2: r' = max(1, round-half-up(r/s))."""
    return _load().fgfo_radius_lowres(r, s)


def subsample(x, s: int, mode: int = NEAREST) -> np.ndarray:
    """Alg. 2 step 1 on one plane."""
    x = _f64(x)
    H, W = x.shape
    out = np.empty((lowres_dim(H, s), lowres_dim(W, s)), np.float64)
    _load().fgfo_subsample(_dptr(x), H, W, s, mode, _dptr(out))
    return out


def box_mean(x, r: int) -> np.ndarray:
    """f_mean(x, r), clip-and-renormalize (R1)."""
    x = _f64(x)
    h, w = x.shape
    out = np.empty_like(x)
    rc = _load().fgfo_box_mean(_dptr(x), h, w, r, _dptr(out))
    if rc:
        raise MemoryError("oracle box_mean failed")
    return out


def upsample(x, H: int, W: int) -> np.ndarray:
    """Bilinear pixel-centre upsample of one plane to H x W (R5)."""
    x = _f64(x)
    h, w = x.shape
    out = np.empty((H, W), np.float64)
    _load().fgfo_upsample(_dptr(x), h, w, H, W, _dptr(out))
    return out


def _shape4(a, C):
    a = _f32(a)
    if a.ndim == 2:
        a = a[None, None]
    elif a.ndim == 3:
        a = a[None] if C == a.shape[0] else a[:, None]
    return np.ascontiguousarray(a)


def coefficients(I, p, r: int, eps: float, s: int, sub_mode: int = NEAREST, with_ab=False):
    """Alg. 2 steps 1-5.  I: [B,C_I,H,W] (or [H,W]), p: [B,C_p,H,W].  Returns the
    low-res mean maps [B, C_p, C_I+1, h, w] (components of mean_a then mean_b), and
    the unsmoothed a, b maps too when with_ab."""
    I = _f32(I)
    p = _f32(p)
    if I.ndim == 2:
        I = I[None, None]
    if p.ndim == 2:
        p = p[None, None]
    B, C_I, H, W = I.shape
    C_p = p.shape[1]
    h, w = lowres_dim(H, s), lowres_dim(W, s)
    mean_ab = np.empty((B, C_p, C_I + 1, h, w), np.float64)
    ab = np.empty_like(mean_ab) if with_ab else None
    rc = _load().fgfo_coefficients(_fptr(I), _fptr(p), B, H, W, C_I, C_p, r, float(eps), s,
                                   sub_mode, _dptr(ab) if with_ab else None, _dptr(mean_ab))
    if rc:
        raise ValueError(f"oracle rejected arguments (rc={rc})")
    return (mean_ab, ab) if with_ab else mean_ab


def upsample_output(I, mean_ab, s: int) -> np.ndarray:
    """Alg. 2 steps 6-7 from given low-res mean maps [B,C_p,C_I+1,h,w]."""
    I = _f32(I)
    if I.ndim == 2:
        I = I[None, None]
    mean_ab = _f64(mean_ab)
    B, C_I, H, W = I.shape
    C_p = mean_ab.shape[1]
    q = np.empty((B, C_p, H, W), np.float64)
    rc = _load().fgfo_upsample_output(_fptr(I), _dptr(mean_ab), _dptr(q), B, H, W, C_I, C_p, s)
    if rc:
        raise ValueError(f"oracle rejected arguments (rc={rc})")
    return q


def fast_guided_filter(I, p, r: int, eps: float, s: int, sub_mode: int = NEAREST) -> np.ndarray:
    """The whole Fast Guided Filter (Alg. 2).  I: [B,C_I,H,W] or [H,W]; p: [B,C_p,H,W] or
    [H,W].  Returns q as float64 [B,C_p,H,W]."""
    I = _f32(I)
    p = _f32(p)
    if I.ndim == 2:
        I = I[None, None]
    if p.ndim == 2:
        p = p[None, None]
    B, C_I, H, W = I.shape
    C_p = p.shape[1]
    if p.shape[0] != B or p.shape[2:] != (H, W):
        raise ValueError("I and p shapes disagree")
    q = np.empty((B, C_p, H, W), np.float64)
    rc = _load().fgfo_filter(_fptr(I), _fptr(p), _dptr(q), B, H, W, C_I, C_p, r, float(eps), s,
                             sub_mode)
    if rc:
        raise ValueError(f"oracle rejected arguments (rc={rc})")
    return q


def guided_filter(I, p, r: int, eps: float) -> np.ndarray:
    """Alg. 1: the s = 1 case of Alg. 2."""
    return fast_guided_filter(I, p, r, eps, 1, NEAREST)


def fast_guided_filter_f64(I, p, r: int, eps: float, s: int, sub_mode: int = NEAREST) -> np.ndarray:
    """Alg. 2 on fp64 inputs (no rounding to fp32): I [B,C_I,H,W], p [B,C_p,H,W]."""
    I = _f64(I)
    p = _f64(p)
    B, C_I, H, W = I.shape
    C_p = p.shape[1]
    if p.shape[0] != B or p.shape[2:] != (H, W):
        raise ValueError("I and p shapes disagree")
    q = np.empty((B, C_p, H, W), np.float64)
    rc = _load().fgfo_filter_f64(_dptr(I), _dptr(p), _dptr(q), B, H, W, C_I, C_p, r, float(eps),
                                 s, sub_mode)
    if rc:
        raise ValueError(f"oracle rejected arguments (rc={rc})")
    return q


def to_grayscale(img) -> np.ndarray:
    """SPEC to_grayscale: luminance 0.299 R + 0.587 G + 0.114 B of a 3-channel image
    [B,3,H,W] (identity for 1 channel), in double: [B,1,H,W]."""
    x = np.asarray(img, dtype=np.float64)
    if x.shape[1] == 1:
        return x.copy()
    if x.shape[1] != 3:
        raise ValueError("to_grayscale takes 1 or 3 channels")
    return (0.299 * x[:, 0] + 0.587 * x[:, 1] + 0.114 * x[:, 2])[:, None]


def enhance(I, gain: float, r: int, eps: float, s: int, sub_mode: int = NEAREST,
            guide: str = "self") -> np.ndarray:
    """Detail enhancement (Fig. 2 caption P:95-97, "enhanced images with x5 detail";
    SPEC S:303-306 enhance): base = the filter of the image (p = I) guided by the image itself
    (guide = "self": colour guidance for RGB, R20) or by its luminance (guide =
    "luma": SPEC's default shared gray guidance, I = to_grayscale(img)), then
    out = (I - base) * gain + base, in double, unclamped."""
    I = _f32(I)
    if I.ndim == 2:
        I = I[None, None]
    if guide == "luma" and I.shape[1] == 3:
        base = fast_guided_filter_f64(to_grayscale(I), I, r, eps, s, sub_mode)
    elif guide in ("self", "luma"):
        base = fast_guided_filter(I, I, r, eps, s, sub_mode)
    else:
        raise ValueError("guide must be 'self' or 'luma'")
    return (I.astype(np.float64) - base) * gain + base


def lowres_chain(Is, ps, r_low: int, eps: float) -> np.ndarray:
    """Alg. 2 steps 2-5 on given low-res planes, all in double: Is [B,C_I,h,w],
    ps [B,C_p,h,w] (any float dtype, widened exactly), radius r_low = r'.  Returns the mean
    maps [B, C_p, C_I+1, h, w]."""
    Is = _f64(Is)
    ps = _f64(ps)
    B, C_I, h, w = Is.shape
    C_p = ps.shape[1]
    if ps.shape[0] != B or ps.shape[2:] != (h, w):
        raise ValueError("I' and p' shapes disagree")
    mean_ab = np.empty((B, C_p, C_I + 1, h, w), np.float64)
    rc = _load().fgfo_lowres_chain(_dptr(Is), _dptr(ps), B, h, w, C_I, C_p, r_low, float(eps),
                                   _dptr(mean_ab))
    if rc:
        raise ValueError(f"oracle rejected arguments (rc={rc})")
    return mean_ab


def joint_upsample(I, p_low, r: int, eps: float, s: int, sub_mode: int = NEAREST) -> np.ndarray:
    """Joint upsampling (R18; the setting P:18 names, no procedure in the paper):
    p is given only at low resolution and IS the p' of Alg. 2; I' = f_sub(I, s), the
    low-res steps run at s = 1 with r' = radius_lowres(r, s), and the output
    uses the full-resolution I.  I: [B,C_I,H,W]; p_low: [B,C_p,h,w] (fp32 or fp64,
    used as given).  Every step is in double: I' is not rounded."""
    I = _f32(I)
    if I.ndim == 2:
        I = I[None, None]
    p_low = _f64(p_low)
    if p_low.ndim == 2:
        p_low = p_low[None, None]
    B, C_I, H, W = I.shape
    Is = np.stack([np.stack([subsample(I[b, c], s, sub_mode) for c in range(C_I)])
                   for b in range(B)])
    if p_low.shape[2:] != Is.shape[2:]:
        raise ValueError("p_low must be [B, C_p, ceil(H/s), ceil(W/s)]")
    mean_ab = lowres_chain(Is, p_low, radius_lowres(r, s), eps)
    return upsample_output(I, mean_ab, s)
