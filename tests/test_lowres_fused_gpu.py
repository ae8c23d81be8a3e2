"""GPU parity of K13, the fused low-res chain for gray guidance (fgf_lowres.cuh), against the
fp64 oracle, with its segment / strip geometry forced small so that every ring wrap, the
top / bottom window clipping and the stage-B warm-up are exercised on small images; and
agreement with the unfused strip engine (K0/K1/K3, FGF_LOWRES=strip) on the same inputs.
"""
from __future__ import annotations

import os

import numpy as np
import pytest
import torch

import oracle

pytestmark = pytest.mark.gpu

import paper_1505_00996_b200 as fgf  # no fallback: a missing libfgf.so fails here


def tol(eps):
    return 1e-4 if eps >= 1e-3 else 1e-3


class env:
    def __init__(self, **kv):
        self.kv = dict(kv, FGF_DEV="1")   # the library honours its development knobs only then

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


def oracle_err(I, p, q, r, eps, s, sub):
    worst = 0.0
    for b in range(I.shape[0]):
        ref = oracle.fast_guided_filter(I[b:b + 1].cpu().numpy(), p[b:b + 1].cpu().numpy(),
                                        r, eps, s, sub)
        got = q[b:b + 1].double().cpu().numpy()
        assert np.isfinite(got).all()
        worst = max(worst, float(np.abs(got - ref).max()))
    return worst


# (B, H, W, C_p, r, eps, s, sub, TH, NT)
CASES = [
    (2, 256, 256, 1, 8, 0.01, 4, 0, None, None),      # config-0 like, default geometry
    (1, 203, 301, 1, 9, 0.01, 4, 0, 8, None),         # many segments, ragged, TH = 2R - 2... 
    (1, 203, 301, 1, 9, 0.01, 4, 0, 5, 128),          # TH not a multiple of G, narrow strips
    (2, 130, 1030, 1, 12, 0.01, 2, 0, 16, 160),       # several strips, R = 6
    (1, 97, 515, 2, 6, 0.02, 3, 1, 7, None),          # block mean, C_p = 2, s = 3
    (1, 64, 64, 1, 60, 0.01, 4, 0, 3, None),          # r' = 15 > low-res size 16
    (1, 50, 70, 2, 3, 1e-5, 1, 0, 9, None),           # s = 1, small eps, C_p = 2
    (3, 1, 300, 1, 2, 0.01, 1, 0, None, None),        # one-row images
    (1, 300, 1, 1, 2, 0.01, 1, 0, 11, None),          # one-column image
    (1, 1024, 1024, 1, 32, 0.01, 4, 0, None, None),   # config-4 geometry (w = 256, R = 8)
]


# kernel variants (fgf_api.cu kLrNumVariants): 0 = sample ring, G 4; 1 = G 8; 2 / 3 = no ring
VARIANTS = [None, "0", "1", "2"]


@pytest.mark.parametrize("variant", VARIANTS)
@pytest.mark.parametrize("case", CASES)
def test_fused_lowres_vs_oracle(case, variant):
    B, H, W, CP, r, eps, s, sub, TH, NT = case
    if variant is not None and CP > 1:
        pytest.skip("one kernel variant for several p channels")
    if variant in ("2", "3"):
        NT = 128 if NT is None else min(NT, 160)
    g = torch.Generator(device="cuda").manual_seed(abs(hash(case)) % (2 ** 31))
    I = torch.rand((B, 1, H, W), device="cuda", generator=g)
    p = torch.rand((B, CP, H, W), device="cuda", generator=g)
    with env(FGF_LR_TH=TH, FGF_LR_NT=NT, FGF_LOWRES=None, FGF_LR_V=variant, FGF_LR_RMAX=64,
             FGF_ENGINE="k13"):
        fgf.fgf_profile_enable(True)
        q = fgf.filter(I, p, r, eps, s, sub)
        torch.cuda.synchronize()
        prof = fgf.fgf_profile_read()
        fgf.fgf_profile_enable(False)
    if variant is not None and prof["lowres_fused"][1] == 0:
        pytest.skip("geometry outside this variant's limits")
    assert prof["lowres_fused"][1] == 1, prof       # the fused kernel served this call
    assert prof["stats_coef"][1] == 0, prof
    err = oracle_err(I, p, q, r, eps, s, sub)
    assert err <= tol(eps), (case, err)


@pytest.mark.parametrize("case", [c for c in CASES if c[0] * c[1] * c[2] <= 1 << 20])
def test_fused_matches_strip_engine(case):
    """Same inputs through K13 and through the unfused K0/K1/K3 strip engine: both are fp64
    box sums of the same fp32 samples, so the mean maps agree to fp32 rounding."""
    B, H, W, CP, r, eps, s, sub, TH, NT = case
    g = torch.Generator(device="cuda").manual_seed(7 + abs(hash(case)) % 1000)
    I = torch.rand((B, 1, H, W), device="cuda", generator=g)
    p = torch.rand((B, CP, H, W), device="cuda", generator=g)
    with env(FGF_LR_TH=TH, FGF_LR_NT=NT, FGF_LOWRES=None, FGF_LR_RMAX=64, FGF_ENGINE="k13"):
        m1 = fgf.coefficients(I, p, r, eps, s, sub)
    with env(FGF_LOWRES="strip"):
        m2 = fgf.coefficients(I, p, r, eps, s, sub)
    torch.cuda.synchronize()
    scale = max(1.0, float(m2.abs().max()))
    assert float((m1 - m2).abs().max()) <= 2e-6 * scale


def test_strip_engine_still_parity_green():
    """The unfused engine stays the path for colour guidance; check it on a gray case too."""
    g = torch.Generator(device="cuda").manual_seed(3)
    I = torch.rand((1, 1, 256, 256), device="cuda", generator=g)
    p = torch.rand((1, 1, 256, 256), device="cuda", generator=g)
    with env(FGF_LOWRES="strip"):
        q = fgf.filter(I, p, 8, 0.01, 4, 0)
        torch.cuda.synchronize()
    assert oracle_err(I, p, q, 8, 0.01, 4, 0) <= 1e-4


def test_tall_image_default_segments():
    """K13 on a 4000-row image: the default geometry caps segments at 512 rows, so
    stage B's fp32 running column sums (R17) take at most 512 add / remove steps; the result
    stays within the oracle tolerance at eps = 1e-3."""
    g = torch.Generator(device="cuda").manual_seed(11)
    I = torch.rand((1, 1, 4000, 96), device="cuda", generator=g)
    p = (I + 0.2 * torch.rand((1, 1, 4000, 96), device="cuda", generator=g)).clamp(0, 1)
    with env(FGF_ENGINE="k13"):
        fgf.fgf_profile_enable(True)
        q = fgf.filter(I, p, 3, 1e-3, 1, 0)
        torch.cuda.synchronize()
        prof = fgf.fgf_profile_read()
        fgf.fgf_profile_enable(False)
    assert prof["lowres_fused"][1] == 1, prof
    assert oracle_err(I, p, q, 3, 1e-3, 1, 0) <= 1e-4


# (B, H, W, r, s, TH): w % 4 == 0 (bulk stores), w % 4 != 0 and TW rounded to 4 columns
BULK_CASES = [
    (2, 1024, 1024, 32, 4, None),     # config-4 geometry: TW 128, every row segment 512 B
    (1, 2160, 3840, 16, 4, None),     # config 1: w = 960, TW rounded 138 -> 140
    (1, 203, 1204, 9, 4, 8),          # w = 301: per-thread stores (no bulk)
    (3, 97, 388, 5, 1, 5),            # s = 1, several segments, ragged last strip
]


@pytest.mark.parametrize("case", BULK_CASES)
def test_bulk_output_stores_bit_identical(case):
    """K13's staged output rows leave by TMA bulk copies when the rows are 16-byte aligned;
    the per-thread store path (FGF_LR_NOBULK) must give the same maps bit for bit (same
    strips: the geometry does not depend on the store path)."""
    B, H, W, r, s, TH = case
    g = torch.Generator(device="cuda").manual_seed(101 + H)
    I = torch.rand((B, 1, H, W), device="cuda", generator=g)
    p = torch.rand((B, 1, H, W), device="cuda", generator=g)
    with env(FGF_LR_TH=TH, FGF_ENGINE="k13", FGF_LR_NOBULK=None):
        fgf.fgf_profile_enable(True)
        m1 = fgf.coefficients(I, p, r, 0.01, s, 0)
        torch.cuda.synchronize()
        prof = fgf.fgf_profile_read()
        fgf.fgf_profile_enable(False)
    with env(FGF_LR_TH=TH, FGF_ENGINE="k13", FGF_LR_NOBULK="1"):
        m2 = fgf.coefficients(I, p, r, 0.01, s, 0)
        torch.cuda.synchronize()
    assert prof["lowres_fused"][1] == 1, prof
    assert torch.equal(m1, m2)
    if (W + s - 1) // s <= 1024 and B * H * W <= 1 << 21:
        q = fgf.filter(I, p, r, 0.01, s, 0)
        torch.cuda.synchronize()
        assert oracle_err(I, p, q, r, 0.01, s, 0) <= 1e-4
