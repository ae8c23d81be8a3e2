"""GPU parity of the detail-enhancement application (Fig. 2)
through fgf_enhance_ws against the fp64 oracle's enhance(), plus its algebraic identities.
The enhancement is folded into the mean maps, so the same two kernels run as for the filter."""
from __future__ import annotations

import numpy as np
import pytest
import torch

import oracle
import synth

pytestmark = pytest.mark.gpu

import paper_1505_00996_b200 as fgf  # no fallback: a missing libfgf.so fails here


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    torch.cuda.set_device(0)
    yield


def tol(eps, gain):
    # the oracle's q error is amplified by |1 - gain| in (I - q) gain + q
    return (1e-4 if eps >= 1e-3 else 1e-3) * max(1.0, abs(1.0 - gain))


@pytest.mark.parametrize("C,H,W,r,eps,s,sub,gain", [
    (1, 540, 960, 16, 0.01, 4, 0, 5.0),       # Fig. 2 preset (r=16, eps=0.1^2, s=4, x5)
    (1, 203, 301, 8, 0.02, 2, 1, 3.0),        # block-mean subsampling, ragged
    (3, 270, 480, 16, 0.01, 4, 0, 5.0),       # colour image (3x3 solve path)
    (1, 256, 256, 8, 0.01, 1, 0, 2.0),        # s = 1: the original guided filter
])
def test_enhance_vs_oracle(C, H, W, r, eps, s, sub, gain):
    g = torch.Generator(device="cuda").manual_seed(C * 1000 + H + s)
    if C == 1:
        I, _ = synth.make_batch(1, "cuda", batch=1, H=H, W=W)
    else:
        I = torch.rand((1, C, H, W), device="cuda", generator=g)
    out = fgf.enhance(I, gain, r, eps, s, sub)
    torch.cuda.synchronize()
    ref = oracle.enhance(I.cpu().numpy(), gain, r, eps, s, sub)
    err = float(np.abs(out.double().cpu().numpy() - ref).max())
    assert err <= tol(eps, gain), err


def test_enhance_identities():
    """gain = 1 returns I bit for bit; gain = 0 is exactly the self-guided filter."""
    I, _ = synth.make_batch(0, "cuda")
    assert torch.equal(fgf.enhance(I, 1.0, 8, 0.01, 4), I)
    assert torch.equal(fgf.enhance(I, 0.0, 8, 0.01, 4), fgf.filter(I, I, 8, 0.01, 4))
    I3 = torch.rand((2, 3, 64, 80), device="cuda")
    assert torch.equal(fgf.enhance(I3, 1.0, 4, 0.01, 2), I3)


def test_enhance_errors():
    I = torch.rand((1, 1, 64, 64), device="cuda")
    out = torch.empty_like(I)
    ws = torch.empty(fgf.fgf_workspace_bytes(1, 64, 64, 1, 1, 8, 4), dtype=torch.uint8,
                     device="cuda")
    st = torch.cuda.current_stream()
    assert fgf.fgf_enhance_ws(I, out, 1, 64, 64, 1, 8, 0.01, 4, 0, -1.0, ws, ws.numel(), st,
                              check=False) == fgf.FGF_ERR_PARAM
    assert fgf.fgf_enhance_ws(I, I, 1, 64, 64, 1, 8, 0.01, 4, 0, 5.0, ws, ws.numel(), st,
                              check=False) == fgf.FGF_ERR_ALIAS
    assert fgf.fgf_enhance_ws(I, out, 1, 64, 64, 2, 8, 0.01, 4, 0, 5.0, ws, ws.numel(), st,
                              check=False) == fgf.FGF_ERR_SHAPE


# ---------------------------------------------------------------- joint upsampling (NEXT-4)

@pytest.mark.parametrize("C_I,C_p,H,W,r,eps,s,sub", [
    (1, 1, 540, 960, 16, 0.01, 4, 0),     # gray (K13 on the low-res planes)
    (3, 1, 300, 400, 60, 1e-6, 4, 0),     # colour guide, one channel (feathering-like)
    (3, 3, 270, 480, 8, 0.01, 4, 1),      # colour, block mean
    (1, 2, 203, 301, 9, 0.02, 3, 1),      # ragged, s = 3
])
def test_joint_upsampling_vs_oracle(C_I, C_p, H, W, r, eps, s, sub):
    g = torch.Generator(device="cuda").manual_seed(C_I * 10 + C_p + H)
    I = torch.rand((2, C_I, H, W), device="cuda", generator=g)
    h, w = -(-H // s), -(-W // s)
    p_low = torch.rand((2, C_p, h, w), device="cuda", generator=g)
    q = fgf.filter_joint(I, p_low, r, eps, s, sub)
    torch.cuda.synchronize()
    ref = oracle.joint_upsample(I.cpu().numpy(), p_low.cpu().numpy(), r, eps, s, sub)
    err = float(np.abs(q.double().cpu().numpy() - ref).max())
    assert err <= (1e-4 if eps >= 1e-3 else 1e-3), err


def test_joint_with_subsampled_p_equals_filter():
    """p_low = f_sub(p) (nearest) makes the joint path the filter itself, bit for bit up to
    the low-res engine's segmentation (same kernels, same samples)."""
    I, p = synth.make_batch(1, "cuda", batch=1, H=540, W=960)
    p_low = p[:, :, ::4, ::4].contiguous()
    q1 = fgf.filter_joint(I, p_low, 16, 0.01, 4, 0)
    q2 = fgf.filter(I, p, 16, 0.01, 4, 0)
    torch.cuda.synchronize()
    assert float((q1 - q2).abs().max()) < 1e-5


@pytest.mark.parametrize("H,W,r,eps,s,sub,gain", [
    (540, 960, 16, 0.01, 4, 0, 5.0),      # Fig. 2 preset on an RGB image
    (203, 301, 8, 0.02, 2, 1, 3.0),       # block mean, ragged
    (128, 160, 6, 0.01, 1, 0, 2.0),       # s = 1
])
def test_enhance_luma_guidance_vs_oracle(H, W, r, eps, s, sub, gain):
    """SPEC enhance with its default shared gray guidance: I = luminance
    0.299 R + 0.587 G + 0.114 B, p = the RGB image (fgf_enhance_ex_ws,
    FGF_GUIDE_LUMA) vs oracle.enhance(guide="luma") in fp64 end to end."""
    g = torch.Generator(device="cuda").manual_seed(H + W + s)
    I = torch.rand((2, 3, H, W), device="cuda", generator=g)
    out = fgf.enhance(I, gain, r, eps, s, sub, guide="luma")
    torch.cuda.synchronize()
    ref = oracle.enhance(I.cpu().numpy(), gain, r, eps, s, sub, guide="luma")
    err = float(np.abs(out.double().cpu().numpy() - ref).max())
    assert err <= tol(eps, gain), err
    # gain = 1: the image itself (to fp32 rounding of gain I + 0 q)
    one = fgf.enhance(I, 1.0, r, eps, s, sub, guide="luma")
    torch.cuda.synchronize()
    assert torch.equal(one, I)
