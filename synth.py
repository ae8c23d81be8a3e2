"""Seeded synthetic inputs for the BASELINE.json configs (stand-ins for the paper's photos).

The paper's test images (Fig. 1-4) are not in the container, so every
input is generated from a seed with the shapes, sizes and value ranges BASELINE.json
names.  This module holds NONE of the filter's arithmetic: it only paints shapes, ramps
and noise.  It is the one module both the CUDA path's tests/bench and the oracle's tests
use.  Recipe:

  seed(cfg, i) = 1_000_003 * cfg + i   (i = global image index; so any sharding of a
                                        batch reproduces the same images)
  shape parameters: numpy.random.default_rng(seed)
  Gaussian noise:   torch.Generator(device).manual_seed(seed)
  all images clamped to [0, 1], stored fp32 planar [B][C][H][W].
"""
from __future__ import annotations

import math

import numpy as np
import torch

NEAREST, BLOCKMEAN = 0, 1

# BASELINE.json configs (W x H there is width x height).
CONFIGS = {
    0: dict(name="cfg0_gray256_selfguided", batch=1, H=256, W=256, C_I=1, C_p=1, r=8, eps=0.01,
            s=4, sub_mode=NEAREST),
    1: dict(name="cfg1_gray_3840x2160", batch=1, H=2160, W=3840, C_I=1, C_p=1, r=16, eps=0.01,
            s=4, sub_mode=NEAREST),
    2: dict(name="cfg2_color_feather_4000x3000", batch=1, H=3000, W=4000, C_I=3, C_p=1, r=60,
            eps=1e-6, s=4, sub_mode=NEAREST),
    3: dict(name="cfg3_color_batch64_1920x1080", batch=64, H=1080, W=1920, C_I=3, C_p=3, r=8,
            eps=0.01, s=4, sub_mode=BLOCKMEAN),
    4: dict(name="cfg4_gray_batch256_4096", batch=256, H=4096, W=4096, C_I=1, C_p=1, r=32,
            eps=0.01, s=4, sub_mode=NEAREST),
    5: dict(name="cfg4b_gray_16384_banded", batch=1, H=16384, W=16384, C_I=1, C_p=1, r=32,
            eps=0.01, s=4, sub_mode=NEAREST),
}


def seed_of(cfg: int, i: int) -> int:
    return 1_000_003 * cfg + i


def _grid(H, W, device):
    ys = torch.arange(H, device=device, dtype=torch.float32).view(H, 1)
    xs = torch.arange(W, device=device, dtype=torch.float32).view(1, W)
    return ys, xs


def _ramp(rng, H, W, device):
    """Linear ramp background 0.2 + 0.6 t, t = (x cos th + y sin th) normalised to [0,1]."""
    th = rng.uniform(0.0, 2.0 * math.pi)
    ys, xs = _grid(H, W, device)
    t = xs * math.cos(th) + ys * math.sin(th)
    t = (t - t.min()) / max(float(t.max() - t.min()), 1e-12)
    return 0.2 + 0.6 * t


def _paint_rect(img, cy, cx, hh, hw, val):
    H, W = img.shape[-2:]
    y0, y1 = max(0, int(round(cy - hh))), min(H, int(round(cy + hh)) + 1)
    x0, x1 = max(0, int(round(cx - hw))), min(W, int(round(cx + hw)) + 1)
    if y0 < y1 and x0 < x1:
        if torch.is_tensor(val):
            img[..., y0:y1, x0:x1] = val.view(-1, 1, 1)
        else:
            img[..., y0:y1, x0:x1] = val


def _paint_ellipse(img, cy, cx, ay, ax, ang, val):
    """Rotated ellipse with semi-axes (ax, ay) rotated by ang, painted only inside its bbox."""
    H, W = img.shape[-2:]
    R = max(ax, ay)
    y0, y1 = max(0, int(cy - R) - 1), min(H, int(cy + R) + 2)
    x0, x1 = max(0, int(cx - R) - 1), min(W, int(cx + R) + 2)
    if y0 >= y1 or x0 >= x1:
        return
    dev = img.device
    ys = torch.arange(y0, y1, device=dev, dtype=torch.float32).view(-1, 1) - cy
    xs = torch.arange(x0, x1, device=dev, dtype=torch.float32).view(1, -1) - cx
    c, s = math.cos(ang), math.sin(ang)
    u = xs * c + ys * s
    v = -xs * s + ys * c
    m = (u / ax) ** 2 + (v / ay) ** 2 <= 1.0
    sub = img[..., y0:y1, x0:x1]
    if torch.is_tensor(val):
        sub.copy_(torch.where(m, val.view(-1, 1, 1), sub))
    else:
        sub.copy_(torch.where(m, torch.full_like(sub, val), sub))


def _noise(gen, shape, sigma, device):
    return torch.randn(shape, generator=gen, device=device, dtype=torch.float32) * sigma


def gray_scene(seed, H, W, device, n_shapes, rects_only=False, noise=0.05):
    """Config 0 / 1 / 4 guidance: shapes (rectangles, or rectangles + rotated ellipses)
    with U[0,1] intensities over a ramp, + N(0, noise^2), clamped (DESIGN.md Inputs)."""
    rng = np.random.default_rng(seed)
    gen = torch.Generator(device=device)
    gen.manual_seed(seed)
    img = _ramp(rng, H, W, device).contiguous()
    for _ in range(n_shapes):
        cy, cx = rng.uniform(0, H), rng.uniform(0, W)
        if rects_only:  # config 0: full side lengths U[W/20, W/4] x U[H/20, H/4]
            sw, sh = rng.uniform(W / 20, W / 4), rng.uniform(H / 20, H / 4)
        else:           # scaled scenes: U[W/40, W/8]
            sw, sh = rng.uniform(W / 40, W / 8), rng.uniform(H / 40, H / 8)
        val = float(rng.uniform(0, 1))
        if not rects_only and rng.uniform() < 0.5:
            _paint_ellipse(img, cy, cx, sh / 2, sw / 2, rng.uniform(0, math.pi), val)
        else:
            _paint_rect(img, cy, cx, sh / 2, sw / 2, val)
    img += _noise(gen, (H, W), noise, device)
    return img.clamp_(0.0, 1.0), gen


def color_scene(seed, H, W, device, n_ellipses=40, noise=0.02):
    """Config 2 / 3 guidance: base colour U[0,1]^3, rotated ellipses with shared geometry and
    per-channel intensities, semi-axes U[W/60, W/6], + independent N(0, noise^2), clamped."""
    rng = np.random.default_rng(seed)
    gen = torch.Generator(device=device)
    gen.manual_seed(seed)
    base = torch.tensor(rng.uniform(0, 1, 3), dtype=torch.float32, device=device)
    img = base.view(3, 1, 1).expand(3, H, W).contiguous()
    for _ in range(n_ellipses):
        cy, cx = rng.uniform(0, H), rng.uniform(0, W)
        ax, ay = rng.uniform(W / 60, W / 6), rng.uniform(W / 60, W / 6)
        ang = rng.uniform(0, math.pi)
        col = torch.tensor(rng.uniform(0, 1, 3), dtype=torch.float32, device=device)
        _paint_ellipse(img, cy, cx, ay, ax, ang, col)
    img += _noise(gen, (3, H, W), noise, device)
    return img.clamp_(0.0, 1.0), rng, gen


def blob_mask(rng, H, W, device, ramp_px=20.0):
    """Config 2 input p: star-shaped blob R(th) = R0 (1 + sum_{k=2..5} c_k cos(k th + phi_k)),
    R0 = 0.25 min(W,H), centre U[0.4,0.6] (W,H); p = clamp(0.5 + (R(th) - d)/ramp_px, 0, 1)."""
    R0 = 0.25 * min(W, H)
    ck = rng.uniform(-0.1, 0.1, 4)
    phik = rng.uniform(0, 2 * math.pi, 4)
    cx, cy = rng.uniform(0.4, 0.6) * W, rng.uniform(0.4, 0.6) * H
    ys, xs = _grid(H, W, device)
    dy, dx = ys - cy, xs - cx
    d = torch.sqrt(dx * dx + dy * dy)
    th = torch.atan2(dy, dx)
    R = torch.ones_like(d)
    for k in range(4):
        R = R + float(ck[k]) * torch.cos((k + 2) * th + float(phik[k]))
    R = R * R0
    return (0.5 + (R - d) / ramp_px).clamp_(0.0, 1.0)


def make_image(cfg: int, i: int, device, H=None, W=None):
    """Image i (global index) of config cfg: returns (I [C_I,H,W], p [C_p,H,W]).
    For config 0 p is I itself (self-guided; the caller may pass the same buffer)."""
    c = CONFIGS[cfg]
    H = H or c["H"]
    W = W or c["W"]
    seed = seed_of(cfg, i)
    if cfg == 0:
        I, _ = gray_scene(seed, H, W, device, 12, rects_only=True, noise=0.05)
        return I.view(1, H, W), I.view(1, H, W)
    if cfg in (1, 4, 5):
        I, gen = gray_scene(seed, H, W, device, 200, rects_only=False, noise=0.05)
        p = (I + _noise(gen, (H, W), 0.1, device)).clamp_(0.0, 1.0)
        return I.view(1, H, W), p.view(1, H, W)
    if cfg == 2:
        I, rng, gen = color_scene(seed, H, W, device)
        return I, blob_mask(rng, H, W, device).view(1, H, W)
    if cfg == 3:
        I, rng, gen = color_scene(seed, H, W, device)
        p = (I + _noise(gen, (3, H, W), 0.05, device)).clamp_(0.0, 1.0)
        return I, p
    raise KeyError(cfg)


def make_batch(cfg: int, device, batch=None, first=0, H=None, W=None):
    """Images [first, first+batch) of config cfg as contiguous fp32 [B,C,H,W] tensors.
    For config 0 the returned p IS I (same storage), as BASELINE.json config 0 states."""
    c = CONFIGS[cfg]
    B = c["batch"] if batch is None else batch
    H = H or c["H"]
    W = W or c["W"]
    I = torch.empty((B, c["C_I"], H, W), dtype=torch.float32, device=device)
    p = I if cfg == 0 else torch.empty((B, c["C_p"], H, W), dtype=torch.float32, device=device)
    for b in range(B):
        Ib, pb = make_image(cfg, first + b, device, H, W)
        I[b].copy_(Ib)
        if cfg != 0:
            p[b].copy_(pb)
    return I, p


def params(cfg: int, **over):
    """Filter parameters of config cfg: dict(r, eps, s, sub_mode), overridable."""
    c = dict(CONFIGS[cfg])
    c.update(over)
    return {k: c[k] for k in ("r", "eps", "s", "sub_mode")}
