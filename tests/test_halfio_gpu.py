"""Reduced-precision I/O: I, p, q stored as float16 / bfloat16 through
fgf_filter_ex_ws.  The oracle receives the 16-bit inputs widened exactly to fp64; the bar is
the fp32 path's tolerance plus half a unit in the last place of the 16-bit q (the only new
rounding is q's store).  A second check pins the 16-bit path to the fp32 path on the same
16-bit-valued inputs: at most one 16-bit rounding step apart."""
from __future__ import annotations

import numpy as np
import pytest
import torch

import oracle
import synth

pytestmark = pytest.mark.gpu

import paper_1505_00996_b200 as fgf  # no fallback: a missing libfgf.so fails here

ULP = {torch.float16: 2.0 ** -10, torch.bfloat16: 2.0 ** -7}   # at magnitudes in [1, 2)


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    torch.cuda.set_device(0)
    yield


CASES = [
    # (cfg-like input, B, C_I, C_p, H, W, r, eps, s, sub)
    ("gray", 2, 1, 1, 1024, 1024, 32, 0.01, 4, 0),    # config 4 geometry (smaller)
    ("gray", 1, 1, 1, 540, 960, 16, 0.01, 1, 0),      # s = 1
    ("gray", 1, 1, 1, 301, 517, 7, 0.02, 3, 1),       # block mean, ragged, odd W
    ("color", 2, 3, 3, 270, 480, 8, 0.01, 4, 1),      # config 3 geometry (smaller)
    ("color", 1, 3, 1, 300, 400, 60, 1e-6, 4, 0),     # config 2 style, eps = 1e-6
]


def _inputs(kind, B, C_I, C_p, H, W, dtype, seed):
    g = torch.Generator(device="cuda").manual_seed(seed)
    if kind == "gray":
        I, p = synth.make_batch(1, "cuda", batch=B, H=H, W=W)
    else:
        I = torch.rand((B, C_I, H, W), device="cuda", generator=g)
        p = (I[:, :C_p] + 0.05 * torch.randn((B, C_p, H, W), device="cuda", generator=g)).clamp(0, 1)
    return I.to(dtype).contiguous(), p.to(dtype).contiguous()


@pytest.mark.parametrize("dtype", [torch.float16, torch.bfloat16])
@pytest.mark.parametrize("case", CASES)
def test_half_io_vs_oracle(case, dtype):
    kind, B, C_I, C_p, H, W, r, eps, s, sub = case
    I, p = _inputs(kind, B, C_I, C_p, H, W, dtype, hash(case) % 1000)
    q = fgf.filter(I, p, r, eps, s, sub)
    torch.cuda.synchronize()
    assert q.dtype == dtype
    base = 1e-4 if eps >= 1e-3 else 1e-3
    for b in range(B):
        ref = oracle.fast_guided_filter(I[b:b + 1].float().cpu().numpy(),
                                        p[b:b + 1].float().cpu().numpy(), r, eps, s, sub)
        got = q[b:b + 1].double().cpu().numpy()
        assert np.isfinite(got).all()
        bound = base + 0.5 * ULP[dtype] * np.maximum(1.0, np.abs(ref))
        assert (np.abs(got - ref) <= bound).all(), float(np.abs(got - ref).max())


@pytest.mark.parametrize("dtype", [torch.float16, torch.bfloat16])
def test_half_io_equals_rounded_fp32_path(dtype):
    I, p = _inputs("gray", 2, 1, 1, 512, 768, dtype, 9)
    q16 = fgf.filter(I, p, 16, 0.01, 4, 0)
    q32 = fgf.filter(I.float().contiguous(), p.float().contiguous(), 16, 0.01, 4, 0)
    torch.cuda.synchronize()
    d = (q16.float() - q32).abs()
    assert float((d - 0.5 * ULP[dtype] * q32.abs().clamp(min=1.0)).max()) <= 1e-6


def test_half_io_unsupported_and_errors():
    I = torch.rand((1, 1, 64, 64), device="cuda").half()
    p = torch.rand((1, 2, 64, 64), device="cuda").half()
    q = torch.empty_like(p)
    ws = torch.empty(1 << 24, dtype=torch.uint8, device="cuda")
    st = torch.cuda.current_stream()
    assert fgf.fgf_filter_ex_ws(I, p, q, 1, 64, 64, 1, 2, 8, 0.01, 4, 0, fgf.FGF_F16, ws,
                                ws.numel(), st, check=False) == fgf.FGF_ERR_UNSUPPORTED
    assert fgf.fgf_filter_ex_ws(I, I, q[:, :1], 1, 64, 64, 1, 1, 8, 0.01, 4, 0, 7, ws,
                                ws.numel(), st, check=False) == fgf.FGF_ERR_PARAM


def test_half_io_multi_chunk_equals_single_chunk(monkeypatch):
    """16-bit buffers through the chunked pipeline (element offsets of 2 bytes)."""
    monkeypatch.setenv("FGF_DEV", "1")   # honour the development knobs
    I, p = _inputs("gray", 6, 1, 1, 1080, 1920, torch.float16, 3)
    monkeypatch.delenv("FGF_CHUNK_MB", raising=False)
    q1 = fgf.filter(I, p, 16, 0.01, 4, 0)
    monkeypatch.setenv("FGF_CHUNK_MB", "1")
    q2 = fgf.filter(I, p, 16, 0.01, 4, 0)
    torch.cuda.synchronize()
    assert torch.equal(q1, q2)
