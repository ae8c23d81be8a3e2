"""Row-band path on the GPU: the stage kernels of libfgf.so driven by the band host logic,
simulated for several ranks in one process (neighbours' planes passed directly; no kernel
waits on another), against the whole-image CUDA path and the oracle."""
from __future__ import annotations

import numpy as np
import pytest
import torch

import oracle
import paper_1505_00996_b200 as fgf
import synth
from paper_1505_00996_b200 import bands

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("C_I,C_p,s,sub,world", [(1, 1, 4, 0, 2), (1, 1, 4, 0, 8), (3, 1, 2, 1, 3),
                                                 (1, 2, 1, 0, 4)])
def test_bands_match_whole_image(C_I, C_p, s, sub, world):
    g = torch.Generator(device="cuda").manual_seed(17 + world)
    H, W, r, eps = 1536, 1032, 32, 0.01
    I = torch.rand((2, C_I, H, W), device="cuda", generator=g)
    p = torch.rand((2, C_p, H, W), device="cuda", generator=g)
    q_whole = fgf.filter(I, p, r, eps, s, sub)
    q_band = bands.filter_bands_local(I, p, r, eps, s, sub, world)
    torch.cuda.synchronize()
    assert float((q_band - q_whole).abs().max()) < 1e-6
    ref = oracle.fast_guided_filter(I[:1].cpu().numpy(), p[:1].cpu().numpy(), r, eps, s, sub)
    assert float(np.abs(q_band[:1].double().cpu().numpy() - ref).max()) < 1e-4


def test_self_guided_bands():
    I, _ = synth.make_batch(0, "cuda", H=512, W=256)
    q = bands.filter_bands_local(I, I, 8, 0.01, 4, 0, 4)
    ref = oracle.fast_guided_filter(I.cpu().numpy(), I.cpu().numpy(), 8, 0.01, 4, 0)
    assert float(np.abs(q.double().cpu().numpy() - ref).max()) < 1e-4


def test_config4b_eight_bands():
    """BASELINE.json config 4b: one 16384^2 image, r=32, s=4, 8 row bands."""
    prm = synth.params(5)
    I, p = synth.make_batch(5, "cuda")
    q_band = bands.filter_bands_local(I, p, prm["r"], prm["eps"], prm["s"], prm["sub_mode"], 8)
    q_whole = fgf.filter(I, p, **prm)
    torch.cuda.synchronize()
    assert float((q_band - q_whole).abs().max()) < 1e-6
    ref = oracle.fast_guided_filter(I.cpu().numpy(), p.cpu().numpy(), **prm)
    assert float(np.abs(q_band.double().cpu().numpy() - ref).max()) < 1e-4


def test_upsample_rows_rejects_missing_maps():
    I = torch.rand((1, 1, 64, 64), device="cuda")
    m = torch.rand((1, 1, 2, 4, 16), device="cuda")
    q = torch.empty_like(I)
    # rows [0, 64) of a 256-row image need low-res rows 0..16, the buffer holds only 0..3
    rc = fgf.fgf_upsample_output_rows(I, m, q, 1, 64, 64, 1, 1, 256, 64, 16, 0, 0, 4, check=False)
    assert rc == fgf.FGF_ERR_PARAM
