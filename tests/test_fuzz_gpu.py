"""Randomised geometry sweep on the GPU against the fp64 oracle: sizes from 1 pixel to a few
hundred, every radius regime (r' from 1 up to beyond the image), every subsampling ratio the
ABI accepts, both subsampling modes, gray / colour guidance with 1-4 p channels, fp32 and
16-bit and 8-bit I/O, self-guidance.  Seeded, so a failure reproduces; FGF_FUZZ_SEEDS=n runs
n seeds instead of 200."""
from __future__ import annotations

import os

import numpy as np
import pytest
import torch

import oracle

pytestmark = pytest.mark.gpu

import paper_1505_00996_b200 as fgf  # no fallback: a missing libfgf.so fails here

HALF_ULP = {torch.float32: 0.0, torch.float16: 2.0 ** -11, torch.bfloat16: 2.0 ** -8}


def _case(seed):
    rng = np.random.default_rng(seed)
    H = int(rng.choice([1, 2, 3, 7, 16, 33, 64, 97, 150, 257, 300]))
    W = int(rng.choice([1, 2, 5, 8, 31, 64, 100, 129, 256, 333, 520]))
    CI = int(rng.choice([1, 3]))
    CP = int(rng.integers(1, 5))
    s = int(rng.integers(1, 9))
    if s > 1 and s >= min(H, W):
        s = 1
    r = int(rng.integers(1, 48))
    eps = float(rng.choice([1e-6, 1e-4, 1e-3, 0.01, 0.2]))
    sub = int(rng.integers(0, 2))
    B = int(rng.integers(1, 3))
    dtype = torch.float32
    if (CI, CP) in ((1, 1), (3, 1), (3, 3)) and rng.random() < 0.3:
        u = rng.random()
        dtype = torch.float16 if u < 1 / 3 else (torch.bfloat16 if u < 2 / 3 else torch.uint8)
    self_guided = CI == 1 and CP == 1 and rng.random() < 0.3
    return B, H, W, CI, CP, r, eps, s, sub, dtype, self_guided


INV255 = torch.tensor(1.0 / 255.0, dtype=torch.float32)   # 8-bit codes decode as k x fl(1/255)


def _store(t, dtype):
    if dtype == torch.uint8:
        return torch.round(t * 255.0).to(torch.uint8).contiguous()
    return t.to(dtype).contiguous()


def _values(t):
    return t.float() * INV255.to(t.device) if t.dtype == torch.uint8 else t.float()


@pytest.mark.parametrize("seed", range(int(os.environ.get("FGF_FUZZ_SEEDS", "200"))))
def test_fuzz_against_oracle(seed):
    B, H, W, CI, CP, r, eps, s, sub, dtype, self_guided = _case(seed)
    g = torch.Generator(device="cuda").manual_seed(1000 + seed)
    I = _store(torch.rand((B, CI, H, W), device="cuda", generator=g), dtype)
    p = I if self_guided else _store(torch.rand((B, CP, H, W), device="cuda", generator=g), dtype)
    q = fgf.filter(I, p, r, eps, s, sub)
    torch.cuda.synchronize()
    tol = 1e-4 if eps >= 1e-3 else 1e-3
    for b in range(B):
        ref = oracle.fast_guided_filter(_values(I[b:b + 1]).cpu().numpy(),
                                        _values(p[b:b + 1]).cpu().numpy(), r, eps, s, sub)
        if dtype == torch.uint8:   # codes: fp32 bound in codes + half a code, vs clamped q
            got = q[b:b + 1].double().cpu().numpy()
            err = np.abs(got - np.clip(ref, 0.0, 1.0) * 255.0)
            assert (err <= 0.5 + 255.0 * tol + 1e-3).all(), (seed, B, H, W, CI, CP, r, eps, s,
                                                             sub, float(err.max()))
            continue
        got = q[b:b + 1].double().cpu().numpy()
        assert np.isfinite(got).all()
        bound = tol + HALF_ULP[dtype] * np.maximum(1.0, np.abs(ref))
        err = np.abs(got - ref)
        assert (err <= bound).all(), (seed, B, H, W, CI, CP, r, eps, s, sub, dtype,
                                      float(err.max()))


@pytest.mark.parametrize("seed", range(int(os.environ.get("FGF_FUZZ_BAND_SEEDS", "40"))))
def test_fuzz_band_loopback(seed):
    """Random row-band splits through the C band path (fgf_filter_bands_loopback: the same
    plans, phases and halo geometry as fgf_filter_band over NCCL) -- overlapped single
    exchange where the bands are tall enough, compacting single or two-step exchange otherwise
    -- against the whole-image filter (same kernels: <= 1e-5) and the oracle."""
    rng = np.random.default_rng(5000 + seed)
    CI = int(rng.choice([1, 3]))
    CP = int(rng.integers(1, 4))
    s = int(rng.choice([1, 2, 3, 4]))
    r = int(rng.integers(2, 40))
    R = max(1, (2 * r + s) // (2 * s))
    mode = int(rng.integers(0, 2))
    nranks = int(rng.integers(2, 7))
    need = (2 * R + 2) if mode == 0 else (R + 2)
    h = int(rng.integers(nranks * need, nranks * need + 200))
    H = min(h * s - int(rng.integers(0, s)), 2400)
    h = -(-H // s)
    need -= int(h * s == H)            # the halo's extra row only when h s != H
    if any((k + 1) * h // nranks - k * h // nranks < need for k in range(nranks)):
        pytest.skip("bands thinner than the exchange depth")
    W = int(rng.integers(max(s + 1, 8), 700))
    sub = int(rng.integers(0, 2))
    eps = float(rng.choice([1e-4, 1e-3, 0.01]))
    g = torch.Generator(device="cuda").manual_seed(6000 + seed)
    I = torch.rand((1, CI, H, W), device="cuda", generator=g)
    p = torch.rand((1, CP, H, W), device="cuda", generator=g)
    nb = fgf.fgf_bands_loopback_workspace_bytes(H, W, CI, CP, r, s, nranks)
    assert nb > 0, (H, W, CI, CP, r, s, nranks)
    ws = torch.empty(nb, dtype=torch.uint8, device="cuda")
    q = torch.empty((1, CP, H, W), device="cuda")
    fgf.fgf_filter_bands_loopback(I, p, q, H, W, CI, CP, r, eps, s, sub, nranks, ws, nb,
                                  torch.cuda.current_stream(), mode=mode)
    q_whole = fgf.filter(I, p, r, eps, s, sub)
    torch.cuda.synchronize()
    assert float((q - q_whole).abs().max()) <= 1e-5, (seed, H, W, CI, CP, r, s, sub, mode, nranks)
    ref = oracle.fast_guided_filter(I.cpu().numpy(), p.cpu().numpy(), r, eps, s, sub)
    assert float(np.abs(q.double().cpu().numpy() - ref).max()) <= 1e-4


@pytest.mark.parametrize("seed", range(int(os.environ.get("FGF_FUZZ_HOST_SEEDS", "40"))))
def test_fuzz_host_entry_point_equals_device(seed):
    """fgf_filter_host_ex on random geometries (the same generator, widths up to 2080 so that
    both the sample-row copy of p and the dense copy occur, H a multiple of s or not, pinned or
    pageable buffers): q is bit-identical to the device entry point on the same values, with
    NaN / 255 planted in the rows of p the method does not read."""
    B, H, W, CI, CP, r, eps, s, sub, dtype, self_guided = _case(seed + 5000)
    rng = np.random.default_rng(seed + 77)
    W = int(rng.choice([W, 512, 1024, 2080]))
    if s > 1 and s >= min(H, W):
        s = 1
    g = torch.Generator(device="cuda").manual_seed(seed)
    I = _store(torch.rand((B, CI, H, W), device="cuda", generator=g), dtype)
    p = I if self_guided else _store(torch.rand((B, CP, H, W), device="cuda", generator=g), dtype)
    qd = fgf.filter(I, p, r, eps, s, sub)
    torch.cuda.synchronize()
    code = {torch.float32: fgf.FGF_F32, torch.float16: fgf.FGF_F16, torch.bfloat16: fgf.FGF_BF16,
            torch.uint8: fgf.FGF_U8}[dtype]
    pin = bool(rng.integers(0, 2))
    Ih = I.cpu()
    ph = Ih if self_guided else p.cpu()
    sparse = fgf.fgf_filter_host_input_bytes(B, H, W, CI, CP, r, s, sub, code, self_guided) < \
        I.element_size() * B * (CI + (0 if self_guided else CP)) * H * W
    if sparse:   # the rows between the sample rows are not read: poison them
        mask = torch.ones(H, dtype=torch.bool)
        mask[::s] = False
        ph[:, :, mask, :] = 255 if dtype == torch.uint8 else float("nan")
    if pin:
        Ih = Ih.pin_memory()
        ph = Ih if self_guided else ph.pin_memory()
    qh = torch.empty(qd.shape, dtype=dtype)
    qh = qh.pin_memory() if pin else qh
    fgf.fgf_filter_host_ex(Ih, ph, qh, B, H, W, CI, CP, r, eps, s, sub, code, 0)
    assert torch.equal(qh, qd.cpu()), (B, H, W, CI, CP, r, eps, s, sub, dtype, self_guided, sparse)
