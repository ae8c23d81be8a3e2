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


# ---------------------------------------------------------------- the C-ABI band path

def _loopback(I, p, r, eps, s, sub, nranks, mode=fgf.FGF_BAND_SINGLE):
    _, C_I, H, W = I.shape
    C_p = p.shape[1]
    q = torch.empty((1, C_p, H, W), device="cuda")
    nb = fgf.fgf_bands_loopback_workspace_bytes(H, W, C_I, C_p, r, s, nranks)
    assert nb > 0
    ws = torch.empty(nb, dtype=torch.uint8, device="cuda")
    fgf.fgf_filter_bands_loopback(I, p, q, H, W, C_I, C_p, r, eps, s, sub, nranks, ws, nb,
                                  torch.cuda.current_stream(), mode=mode)
    torch.cuda.synchronize()
    return q


@pytest.mark.parametrize("mode", [0, 1])   # FGF_BAND_SINGLE, FGF_BAND_TWO_STEP
@pytest.mark.parametrize("C_I,C_p,s,sub,nranks", [(1, 1, 4, 0, 1), (1, 1, 4, 0, 2), (1, 1, 4, 0, 8),
                                                  (3, 1, 2, 1, 3), (1, 2, 1, 0, 4), (3, 3, 4, 0, 5)])
def test_c_band_loopback_matches_whole_image(C_I, C_p, s, sub, nranks, mode):
    """fgf_filter_bands_loopback: the C band path (same plan, subsample, halo geometry and
    finish as fgf_filter_band; halos copied between the bands' buffers) against the
    whole-image filter and the oracle."""
    g = torch.Generator(device="cuda").manual_seed(23 + nranks)
    H, W, r, eps = 1200, 1032, 32, 0.01
    I = torch.rand((1, C_I, H, W), device="cuda", generator=g)
    p = torch.rand((1, C_p, H, W), device="cuda", generator=g)
    q = _loopback(I, p, r, eps, s, sub, nranks, mode)
    q_whole = fgf.filter(I, p, r, eps, s, sub)
    torch.cuda.synchronize()
    assert float((q - q_whole).abs().max()) < 1e-5
    ref = oracle.fast_guided_filter(I.cpu().numpy(), p.cpu().numpy(), r, eps, s, sub)
    assert float(np.abs(q.double().cpu().numpy() - ref).max()) < 1e-4


@pytest.mark.parametrize("mode", [0, 1])
def test_c_band_loopback_self_guided_config4b_shape(mode):
    I, _ = synth.make_batch(0, "cuda", H=2048, W=512)
    q = _loopback(I, I, 32, 0.01, 4, 0, 8, mode)
    ref = oracle.fast_guided_filter(I.cpu().numpy(), I.cpu().numpy(), 32, 0.01, 4, 0)
    assert float(np.abs(q.double().cpu().numpy() - ref).max()) < 1e-4


def test_c_band_single_rank_with_nccl_communicator():
    """fgf_filter_band through a real (one-rank) NCCL communicator: NCCL loads, the
    communicator initialises, and the band equals the whole-image filter."""
    uid = fgf.fgf_nccl_unique_id()
    comm = fgf.fgf_nccl_comm_init(uid, 0, 1)
    try:
        g = torch.Generator(device="cuda").manual_seed(5)
        H, W = 640, 480
        I = torch.rand((1, 1, H, W), device="cuda", generator=g)
        p = torch.rand((1, 1, H, W), device="cuda", generator=g)
        q = torch.empty_like(p)
        nb = fgf.fgf_band_workspace_bytes(H, W, 0, H, 1, 1, 16, 4, 1)
        ws = torch.empty(nb, dtype=torch.uint8, device="cuda")
        fgf.fgf_filter_band(I, p, q, H, W, 0, H, 1, 1, 16, 0.01, 4, 0, comm, 0, 1, ws, nb,
                            torch.cuda.current_stream())
        torch.cuda.synchronize()
        assert float((q - fgf.filter(I, p, 16, 0.01, 4, 0)).abs().max()) < 1e-5
        q2 = torch.empty_like(p)
        fgf.fgf_filter_band_ex(I, p, q2, H, W, 0, H, 1, 1, 16, 0.01, 4, 0,
                               fgf.FGF_BAND_TWO_STEP, comm, 0, 1, ws, nb,
                               torch.cuda.current_stream())
        torch.cuda.synchronize()
        assert float((q2 - q).abs().max()) < 1e-5
        assert fgf.fgf_nccl_check(comm) == fgf.FGF_OK
    finally:
        fgf.fgf_nccl_comm_destroy(comm)


def test_c_band_errors():
    I = torch.rand((1, 1, 64, 64), device="cuda")
    q = torch.empty_like(I)
    ws = torch.empty(1 << 22, dtype=torch.uint8, device="cuda")
    st = torch.cuda.current_stream()
    # a band thinner than the 2r'+1-row halo, with several ranks
    assert fgf.fgf_filter_band(I, I, q, 256, 64, 0, 64, 1, 1, 32, 0.01, 4, 0, None, 0, 4, ws,
                               ws.numel(), st, check=False) == fgf.FGF_ERR_PARAM
    # several ranks and no communicator
    assert fgf.fgf_filter_band(I, I, q, 1024, 64, 0, 64, 1, 1, 4, 0.01, 4, 0, None, 0, 4, ws,
                               ws.numel(), st, check=False) == fgf.FGF_ERR_NULL
    # row0 not on the subsample grid
    assert fgf.fgf_filter_band(I, I, q, 1024, 64, 2, 64, 1, 1, 4, 0.01, 4, 0, None, 0, 1, ws,
                               ws.numel(), st, check=False) == fgf.FGF_ERR_PARAM


@pytest.mark.parametrize("mode", [0, 1])
@pytest.mark.parametrize("H,W,s,r,nranks", [(1003, 517, 4, 16, 3), (641, 300, 3, 9, 5),
                                            (400, 128, 1, 6, 4), (1024, 200, 8, 40, 2)])
def test_c_band_uneven_splits(H, W, s, r, nranks, mode):
    """Bands of unequal heights, a last band ending off the subsample grid, s = 1 and s = 8,
    r' from 2 to 6: the loop-back band path equals the whole-image filter."""
    g = torch.Generator(device="cuda").manual_seed(H + W + nranks)
    I = torch.rand((1, 1, H, W), device="cuda", generator=g)
    p = torch.rand((1, 1, H, W), device="cuda", generator=g)
    q = _loopback(I, p, r, 0.01, s, 0, nranks, mode)
    q_whole = fgf.filter(I, p, r, 0.01, s, 0)
    torch.cuda.synchronize()
    assert float((q - q_whole).abs().max()) < 1e-5


def test_c_band_loopback_two_step_narrow_bands():
    """Bands of r'+1 <= rows < 2r'+1 low-res rows (here 12-13 rows at r' = 8): only the
    two-step exchange admits them.  The workspace query must still size them."""
    g = torch.Generator(device="cuda").manual_seed(41)
    H, W, r, s, eps, nranks = 2048, 256, 32, 4, 0.01, 40
    I = torch.rand((1, 1, H, W), device="cuda", generator=g)
    p = torch.rand((1, 1, H, W), device="cuda", generator=g)
    assert fgf.fgf_band_workspace_bytes(H, W, 0, 48, 1, 1, r, s, nranks) > 0
    q = _loopback(I, p, r, eps, s, 0, nranks, fgf.FGF_BAND_TWO_STEP)
    ref = oracle.fast_guided_filter(I.cpu().numpy(), p.cpu().numpy(), r, eps, s, 0)
    assert float(np.abs(q.double().cpu().numpy() - ref).max()) < 1e-4
    # the single exchange rejects such bands before any launch
    q2 = torch.empty_like(q)
    nb = fgf.fgf_bands_loopback_workspace_bytes(H, W, 1, 1, r, s, nranks)
    ws = torch.empty(nb, dtype=torch.uint8, device="cuda")
    rc = fgf.fgf_filter_bands_loopback(I, p, q2, H, W, 1, 1, r, eps, s, 0, nranks, ws, nb,
                                       torch.cuda.current_stream(), mode=fgf.FGF_BAND_SINGLE,
                                       check=False)
    assert rc == fgf.FGF_ERR_PARAM


@pytest.mark.parametrize("sub", [0, 1])
def test_c_band_block_mean_workspace(sub):
    """Found by the band fuzz (seed 11): with the block mean (R4) a band's own chain needs the
    compact I', p' planes, which the workspace query sized for the nearest mode only (NOMEM).
    The query now covers both subsampling modes, as fgf_workspace_bytes does."""
    H, W, CI, CP, r, s, nranks = 560, 119, 1, 2, 14, 4, 4
    g = torch.Generator(device="cuda").manual_seed(11)
    I = torch.rand((1, CI, H, W), device="cuda", generator=g)
    p = torch.rand((1, CP, H, W), device="cuda", generator=g)
    q = _loopback(I, p, r, 1e-3, s, sub, nranks, fgf.FGF_BAND_SINGLE)
    q_whole = fgf.filter(I, p, r, 1e-3, s, sub)
    torch.cuda.synchronize()
    assert float((q - q_whole).abs().max()) <= 1e-5


@pytest.mark.parametrize("mode", [0, 1])
@pytest.mark.parametrize("H,s,sub,nranks", [(253, 4, 1, 6), (253, 4, 0, 8), (1021, 8, 0, 5),
                                            (2045, 4, 1, 3)])
def test_c_band_height_not_a_multiple_of_s(H, s, sub, nranks, mode):
    """Found by the band fuzz (seed 153): when h s != H the map scale h / H exceeds 1 / s and
    the last rows of a band upsample from the low-res row after the band, so the halo carries
    one more row (fgf_band.cuh).  Before the fix row 211 of this 253-row image was off by 2e-3."""
    W, r, eps = 364, 2 * s, 1e-3
    g = torch.Generator(device="cuda").manual_seed(H + nranks)
    I = torch.rand((1, 1, H, W), device="cuda", generator=g)
    p = torch.rand((1, 2, H, W), device="cuda", generator=g)
    q = _loopback(I, p, r, eps, s, sub, nranks, mode)
    q_whole = fgf.filter(I, p, r, eps, s, sub)
    torch.cuda.synchronize()
    assert float((q - q_whole).abs().max()) <= 1e-5
