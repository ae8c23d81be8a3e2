"""K5 (csrc/fgf_wide.cuh): the radius-independent fused engine for gray guidance -- the exact
guided filter (Alg. 1) in one kernel at s = 1, and the low-res chain of
Alg. 2 for wide windows r' at s > 1 -- against the fp64 oracle, at sizes that span
several strips, segments, persistent-grid rounds and ragged tails, plus the edge cases
(windows wider than the image, one-row / one-column images, radius 2 = the smallest K5
takes: 4).  Bar: 1e-4 for eps >= 1e-3, 1e-3 below (R15)."""
from __future__ import annotations

import os

import numpy as np
import pytest
import torch

import oracle
import paper_1505_00996_b200 as fgf
import synth

pytestmark = pytest.mark.gpu


def tol(eps):
    return 1e-4 if eps >= 1e-3 else 1e-3


class env:
    """Development knobs of the library (honoured with FGF_DEV=1)."""

    def __init__(self, **kv):
        self.kv = dict(kv, FGF_DEV="1")

    def __enter__(self):
        self.old = {k: os.environ.get(k) for k in self.kv}
        for k, v in self.kv.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = str(v)

    def __exit__(self, *a):
        for k, v in self.old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v


def profiled(fn):
    """Run fn with the library's per-kernel events on; return (result, {kind: launches})."""
    fgf.fgf_profile_enable(True)
    out = fn()
    torch.cuda.synchronize()
    prof = fgf.fgf_profile_read()
    fgf.fgf_profile_enable(False)
    return out, {k: v[1] for k, v in prof.items() if v[1]}


def oracle_err(I, p, q, r, eps, s, sub_mode, images=None):
    sub = sub_mode
    worst = 0.0
    for b in (range(I.shape[0]) if images is None else images):
        ref = oracle.fast_guided_filter(I[b:b + 1].cpu().numpy(), p[b:b + 1].cpu().numpy(), r,
                                        eps, s, sub)
        got = q[b:b + 1].double().cpu().numpy()
        assert np.isfinite(got).all()
        worst = max(worst, float(np.abs(got - ref).max()))
    return worst


# ---------------------------------------------------------------- Alg. 1 (s = 1), one kernel

@pytest.mark.parametrize("B,H,W,r,eps", [
    (1, 257, 333, 16, 0.01),       # ragged, one strip per image width
    (2, 300, 1100, 32, 0.01),      # several strips (TW <= 672 - 4r)
    (1, 96, 700, 4, 0.01),         # the smallest radius K5 takes (ring of 2r+1 >= 8 rows)
    (1, 130, 150, 60, 1e-6),       # window wider than half the image, eps class 1e-3
    (3, 64, 64, 40, 0.04),         # window covers the whole image
    (1, 1, 517, 5, 0.01),          # one row
    (1, 411, 1, 7, 0.01),          # one column
    (1, 5, 9, 4, 0.01),            # tiny
])
def test_exact_guided_filter_one_kernel(B, H, W, r, eps):
    g = torch.Generator(device="cuda").manual_seed(H * 7 + W + r)
    I = torch.rand((B, 1, H, W), device="cuda", generator=g)
    p = torch.rand((B, 1, H, W), device="cuda", generator=g)
    with env(FGF_ENGINE="wide"):                    # (small images default to K6)
        q, kinds = profiled(lambda: fgf.filter(I, p, r, eps, 1, 0))
    assert kinds == {"wide_fused": 1}, kinds        # Alg. 1 is ONE launch: q written directly
    assert oracle_err(I, p, q, r, eps, 1, 0) <= tol(eps)
    with env(FGF_ENGINE="wide", FGF_WIDE_BULK=1):   # TMA bulk staging of the sample rows
        qb = fgf.filter(I, p, r, eps, 1, 0)
    torch.cuda.synchronize()
    assert float((qb - q).abs().max()) == 0.0


@pytest.mark.parametrize("V", ["0", "1", "2"])
@pytest.mark.parametrize("TW,SEGS,GRID", [(32, 7, None), (96, 3, 2), (200, 1, 1), (64, 40, 5),
                                          (301, 2, 3)])
def test_exact_guided_filter_geometries(TW, SEGS, GRID, V):
    """Forced strip widths, segment counts and persistent-grid sizes (several items per CTA,
    segment borders inside windows, ragged last strip / segment), in both kernel variants
    (8-row batches, one CTA per SM: the default at s = 1; 4-row batches, two per SM: the
    mean-maps default): same q as the default geometry within rounding, and within
    tolerance of the oracle."""
    I, p = synth.make_batch(1, "cuda", batch=2, H=203, W=301)
    r, eps = 9, 0.01
    q0 = fgf.filter(I, p, r, eps, 1, 0)
    with env(FGF_WIDE_TW=TW, FGF_WIDE_SEGS=SEGS, FGF_WIDE_GRID=GRID, FGF_WIDE_V=V):
        q1 = fgf.filter(I, p, r, eps, 1, 0)
    torch.cuda.synchronize()
    assert float((q0 - q1).abs().max()) <= 2e-6
    assert oracle_err(I, p, q1, r, eps, 1, 0) <= 1e-4


def test_config1_full_resolution():
    """BASELINE.json config 1 at s = 1 (3840 x 2160, r = 16): the exact guided filter."""
    prm = synth.params(1, s=1)
    I, p = synth.make_batch(1, "cuda")
    q, kinds = profiled(lambda: fgf.filter(I, p, **prm))
    assert kinds == {"wide_fused": 1}, kinds
    assert oracle_err(I, p, q, **prm) <= 1e-4


def test_config4_full_resolution_sampled():
    """BASELINE.json config 4 at s = 1 (r = 32) in the bench's launch configuration (32 of its
    4096^2 images in one call): the oracle on sampled images."""
    prm = synth.params(4, s=1)
    I, p = synth.make_batch(4, "cuda", batch=32)
    q = fgf.filter(I, p, **prm)
    torch.cuda.synchronize()
    assert oracle_err(I, p, q, **prm, images=[0, 31]) <= 1e-4


def test_self_guided_and_tall():
    """p = I (config 0's self-guidance) and a tall image (4000 rows in one segment): the fp64
    vertical running sums do not drift with the height."""
    g = torch.Generator(device="cuda").manual_seed(3)
    I = torch.rand((1, 1, 4000, 64), device="cuda", generator=g)
    with env(FGF_WIDE_SEGS=1):
        q = fgf.filter(I, I, 12, 1e-3, 1, 0)
    torch.cuda.synchronize()
    assert oracle_err(I, I, q, 12, 1e-3, 1, 0) <= 1e-4


@pytest.mark.parametrize("dt", [torch.float16, torch.bfloat16, torch.uint8])
def test_exact_guided_filter_reduced_precision_io(dt):
    """16-bit and 8-bit I/O at s = 1 (K5 reads and writes the elements itself): the oracle fed
    the decoded inputs; bar = fp32 tolerance + half an element ulp of q."""
    g = torch.Generator(device="cuda").manual_seed(5)
    I = torch.rand((2, 1, 200, 260), device="cuda", generator=g)
    p = (I + 0.1 * torch.randn(I.shape, device="cuda", generator=g)).clamp(0, 1)
    if dt == torch.uint8:
        enc = lambda t: torch.round(t * 255).to(torch.uint8)
        dec = lambda t: t.float() * np.float32(1.0 / 255.0)
        half_ulp = 0.5 / 255 + 1e-6
    else:
        enc = lambda t: t.to(dt)
        dec = lambda t: t.float()
        half_ulp = 2.0 ** -9 if dt == torch.bfloat16 else 2.0 ** -12
    Ie, pe = enc(I).contiguous(), enc(p).contiguous()
    q, kinds = profiled(lambda: fgf.filter(Ie, pe, 16, 0.01, 1, 0))
    assert kinds == {"wide_fused": 1}, kinds
    Id, pd = dec(Ie), dec(pe)
    ref = oracle.fast_guided_filter(Id.cpu().numpy(), pd.cpu().numpy(), 16, 0.01, 1, 0)
    if dt == torch.uint8:
        ref = np.clip(ref, 0.0, 1.0)
    err = float(np.abs(dec(q).double().cpu().numpy() - ref).max())
    assert err <= 1e-4 + 1.01 * half_ulp * (2.0 if dt != torch.uint8 else 1.0), err


def test_enhance_at_full_resolution():
    """Detail enhancement (the K13/K3 gain fold) through K5 at s = 1."""
    g = torch.Generator(device="cuda").manual_seed(9)
    I = torch.rand((1, 1, 180, 240), device="cuda", generator=g)
    out = fgf.enhance(I, gain=5.0, r=8, eps=0.01, s=1)
    torch.cuda.synchronize()
    ref = oracle.enhance(I.cpu().numpy(), 5.0, 8, 0.01, 1, 0)
    assert float(np.abs(out.double().cpu().numpy() - ref).max()) <= 4 * 1e-4


# ---------------------------------------------------------------- low-res chain (s > 1)

@pytest.mark.parametrize("H,W,r,s,sub,eps", [
    (1024, 1024, 32, 2, 0, 0.01),     # config 4's s = 2 geometry (r' = 16), one image
    (777, 1203, 60, 4, 0, 1e-6),      # r' = 15, ragged, eps class 1e-3
    (600, 800, 40, 2, 1, 0.01),       # block-mean samples (K0 planes), r' = 20
    (203, 301, 13, 1, 0, 0.01),       # s = 1 maps through fgf_coefficients below
])
def test_wide_lowres_chain(H, W, r, s, sub, eps):
    g = torch.Generator(device="cuda").manual_seed(H + W + r + s)
    I = torch.rand((2, 1, H, W), device="cuda", generator=g)
    p = torch.rand((2, 1, H, W), device="cuda", generator=g)
    with env(FGF_ENGINE="wide"):
        q, kinds = profiled(lambda: fgf.filter(I, p, r, eps, s, sub))
        m = fgf.coefficients(I, p, r, eps, s, sub)
    torch.cuda.synchronize()
    assert "wide_fused" in kinds, kinds
    assert oracle_err(I, p, q, r, eps, s, sub) <= tol(eps)
    ref = oracle.coefficients(I[:1].cpu().numpy(), p[:1].cpu().numpy(), r, eps, s, sub)
    # mean maps: fp32 a, b (R13) -> relative to the largest |mean_a|, |mean_b|
    scale = max(1.0, float(np.abs(ref).max()))
    assert float(np.abs(m[:1].double().cpu().numpy() - ref).max()) <= 2e-5 * scale


@pytest.mark.parametrize("r,s", [(16, 4), (32, 8), (24, 4)])
def test_wide_agrees_with_k13(r, s):
    """Where K13 also applies (r' <= 12): K5 and K13 compute the same maps up to fp32 rounding
    of a, b and of K13's fp32 stage-B sums (R17)."""
    I, p = synth.make_batch(4, "cuda", batch=2, H=1024, W=768)
    with env(FGF_ENGINE="wide"):
        mw = fgf.coefficients(I, p, r, 0.01, s, 0)
    with env(FGF_ENGINE="k13"):
        mk = fgf.coefficients(I, p, r, 0.01, s, 0)
    torch.cuda.synchronize()
    assert float((mw - mk).abs().max()) <= 2e-5
