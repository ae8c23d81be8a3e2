"""GPU parity of the CUDA path (through the C ABI) against the fp64 CPU oracle.

Bar (BASELINE.json north_star): max|q_gpu - q_oracle| <= 1e-4 when eps >= 1e-3 and
<= 1e-3 when eps < 1e-3 (R15), images in [0,1].  Inputs are the seeded synthetic
stand-ins of synth.py; the oracle receives host copies of exactly the GPU's fp32 inputs.
"""
from __future__ import annotations

import numpy as np
import pytest
import torch

import oracle
import synth

pytestmark = pytest.mark.gpu

import paper_1505_00996_b200 as fgf  # no fallback: a missing libfgf.so fails here


def tol(eps):
    return 1e-4 if eps >= 1e-3 else 1e-3


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    torch.cuda.set_device(0)
    yield


def gpu_filter(I, p, r, eps, s, sub_mode):
    q = fgf.filter(I, p, r, eps, s, sub_mode)
    torch.cuda.synchronize()
    # K13 (or K0/K1/K3) + K4, or K5 / K6 alone, went through libfgf.so
    assert fgf.fgf_last_launch_count() >= 1
    return q


def compare(I, p, q, r, eps, s, sub_mode, images=None):
    """Oracle on the listed images (all by default); returns the max abs error."""
    B = I.shape[0]
    images = range(B) if images is None else images
    worst = 0.0
    for b in images:
        Ih = I[b:b + 1].cpu().numpy()
        ph = p[b:b + 1].cpu().numpy()
        ref = oracle.fast_guided_filter(Ih, ph, r, eps, s, sub_mode)
        got = q[b:b + 1].double().cpu().numpy()
        assert np.isfinite(got).all()
        worst = max(worst, float(np.abs(got - ref).max()))
    return worst


# ---------------------------------------------------------------- BASELINE.json configs

@pytest.mark.parametrize("cfg", [0, 1, 2])
def test_config_single_image(cfg):
    prm = synth.params(cfg)
    I, p = synth.make_batch(cfg, "cuda")
    q = gpu_filter(I, p, **prm)
    err = compare(I, p, q, **prm)
    assert err <= tol(prm["eps"]), err


def test_config1_s1_exact_guided_filter():
    prm = synth.params(1, s=1)
    I, p = synth.make_batch(1, "cuda")
    q = gpu_filter(I, p, **prm)
    err = compare(I, p, q, **prm)
    assert err <= tol(prm["eps"]), err


def test_config3_full_batch_sampled():
    """Config 3 in the bench launch configuration (64 images, one call); oracle on a
    deterministic sample of images."""
    prm = synth.params(3)
    I, p = synth.make_batch(3, "cuda")
    q = gpu_filter(I, p, **prm)
    err = compare(I, p, q, **prm, images=[0, 1, 31, 63])
    assert err <= tol(prm["eps"]), err


@pytest.mark.parametrize("s", [4])
def test_config4_full_batch_sampled(s):
    """Config 4 (256 x 4096^2) exactly as bench.py runs it; oracle on images 0, 1, 127, 255."""
    prm = synth.params(4, s=s)
    I, p = synth.make_batch(4, "cuda")
    q = gpu_filter(I, p, **prm)
    err = compare(I, p, q, **prm, images=[0, 1, 127, 255])
    assert err <= tol(prm["eps"]), err


@pytest.mark.parametrize("s", [1, 2, 8])
def test_config4_s_sweep(s):
    prm = synth.params(4, s=s)
    I, p = synth.make_batch(4, "cuda", batch=2)
    q = gpu_filter(I, p, **prm)
    err = compare(I, p, q, **prm)
    assert err <= tol(prm["eps"]), err


# ---------------------------------------------------------------- ragged / edge geometry

CASES = [
    # (B, H, W, C_I, C_p, r, eps, s, sub)
    (2, 37, 53, 1, 1, 3, 0.01, 4, 0),      # ragged low-res, W % 4 != 0 (scalar output path)
    (1, 301, 517, 1, 2, 7, 0.02, 3, 1),    # s = 3, block mean with partial blocks, C_p = 2
    (3, 64, 100, 3, 1, 5, 1e-4, 2, 0),     # color, small eps
    (1, 97, 1031, 3, 4, 9, 0.01, 4, 1),    # color, C_p = 4, w > 256 (several strips)
    (1, 200, 2052, 1, 3, 16, 0.01, 2, 0),  # w = 1026: several strips with halos
    (1, 1, 130, 1, 1, 2, 0.01, 1, 0),      # one-row image, s = 1 (R7)
    (1, 130, 1, 1, 1, 2, 0.01, 1, 0),      # one-column image
    (2, 16, 16, 1, 1, 60, 0.01, 4, 0),     # r' larger than the low-res image
    (1, 40, 44, 1, 1, 1, 0.01, 4, 0),      # s > r: r' clipped to 1
    (1, 120, 2048, 1, 1, 150, 0.01, 1, 0), # r' = 150: 512-thread strips
    (1, 300, 700, 3, 1, 100, 1e-6, 1, 0),  # color, large r', NT = 512 single strip
    (1, 33, 4097, 1, 1, 4, 0.05, 8, 1),    # s = 8 block mean, ragged
    (4, 128, 128, 1, 4, 8, 0.01, 4, 0),    # gray, 4 p channels, batch
    (1, 5, 7, 3, 3, 2, 0.01, 2, 1),        # tiny
]


@pytest.mark.parametrize("case", CASES)
def test_ragged_and_edge_cases(case):
    B, H, W, CI, CP, r, eps, s, sub = case
    g = torch.Generator(device="cuda").manual_seed(hash(case) % (2 ** 31))
    I = torch.rand((B, CI, H, W), device="cuda", generator=g)
    p = torch.rand((B, CP, H, W), device="cuda", generator=g)
    q = gpu_filter(I, p, r, eps, s, sub)
    err = compare(I, p, q, r, eps, s, sub)
    assert err <= tol(eps), (case, err)


def test_self_guided_aliasing():
    """I == p (config 0 style) must equal the result with a separate copy of p."""
    I, _ = synth.make_batch(0, "cuda")
    q1 = gpu_filter(I, I, 8, 0.01, 4, 0)
    q2 = gpu_filter(I, I.clone(), 8, 0.01, 4, 0)
    assert torch.equal(q1, q2)


# ---------------------------------------------------------------- stages in isolation

@pytest.mark.parametrize("CI,CP,s,sub", [(1, 1, 4, 0), (3, 3, 4, 1), (3, 1, 2, 0), (1, 2, 1, 0)])
def test_stage_coefficients(CI, CP, s, sub):
    """Stages 1-5 (fgf_coefficients) against the oracle's mean maps."""
    g = torch.Generator(device="cuda").manual_seed(5 + CI + CP + s)
    I = torch.rand((2, CI, 203, 301), device="cuda", generator=g)
    p = torch.rand((2, CP, 203, 301), device="cuda", generator=g)
    m = fgf.coefficients(I, p, 9, 0.01, s, sub)
    torch.cuda.synchronize()
    ref = oracle.coefficients(I.cpu().numpy(), p.cpu().numpy(), 9, 0.01, s, sub)
    assert m.shape == ref.shape
    assert float(np.abs(m.double().cpu().numpy() - ref).max()) < 2e-5


@pytest.mark.parametrize("CI,CP,s,H,W", [(1, 1, 4, 256, 256), (3, 3, 4, 270, 480),
                                         (1, 2, 3, 101, 203), (3, 1, 1, 64, 64),
                                         (1, 1, 8, 1000, 1024)])
def test_stage_upsample_output(CI, CP, s, H, W):
    """Stages 6-7 alone (K4), fed with oracle-produced mean maps rounded to fp32; the oracle
    gets the same fp32 maps, so this isolates the upsample + output kernel."""
    rng = np.random.default_rng(CI * 100 + CP * 10 + s)
    I = rng.random((2, CI, H, W)).astype(np.float32)
    p = rng.random((2, CP, H, W)).astype(np.float32)
    m = oracle.coefficients(I, p, 8, 0.01, s, 0).astype(np.float32)
    q = fgf.upsample_output(torch.from_numpy(I).cuda(), torch.from_numpy(m).cuda(), s)
    torch.cuda.synchronize()
    ref = oracle.upsample_output(I, m.astype(np.float64), s)
    assert float(np.abs(q.double().cpu().numpy() - ref).max()) < 2e-6


# ---------------------------------------------------------------- identities, robustness

@pytest.mark.parametrize("CI,s,sub", [(1, 4, 0), (3, 4, 1), (3, 1, 0)])
def test_constant_p(CI, s, sub):
    g = torch.Generator(device="cuda").manual_seed(11)
    I = torch.rand((1, CI, 300, 400), device="cuda", generator=g)
    p = torch.full((1, 2, 300, 400), 0.3, device="cuda")
    p[:, 1] = 0.8
    q = gpu_filter(I, p, 16, 1e-6, s, sub)
    assert float((q[:, 0] - 0.3).abs().max()) < 1e-5
    assert float((q[:, 1] - 0.8).abs().max()) < 1e-5


def test_noise_free_color_feathering_robustness():
    """noise-free piecewise-constant colour guidance makes Sigma singular
    (rank 0 in flat windows); fp64 statistics + solve must stay within 1e-3 at eps=1e-6."""
    I, rng, _ = synth.color_scene(synth.seed_of(2, 99), 750, 1000, "cuda", noise=0.0)
    p = synth.blob_mask(rng, 750, 1000, "cuda").view(1, 1, 750, 1000)
    I = I.view(1, 3, 750, 1000).contiguous()
    q = gpu_filter(I, p, 60, 1e-6, 4, 0)
    err = compare(I, p, q, 60, 1e-6, 4, 0)
    assert err <= 1e-3, err


def test_deterministic_and_batch_split_invariant():
    """P16: bitwise identical results across runs and however the batch is split."""
    I, p = synth.make_batch(3, "cuda", batch=4, H=270, W=480)
    prm = synth.params(3)
    q1 = gpu_filter(I, p, **prm)
    q2 = gpu_filter(I, p, **prm)
    assert torch.equal(q1, q2)
    for b in range(4):
        qb = gpu_filter(I[b:b + 1].contiguous(), p[b:b + 1].contiguous(), **prm)
        assert torch.equal(qb, q1[b:b + 1])


def test_host_entry_point_matches_device():
    I, p = synth.make_batch(1, "cuda", batch=3, H=540, W=960)
    prm = synth.params(1)
    qd = gpu_filter(I, p, **prm)
    Ih, ph = I.cpu().pin_memory(), p.cpu().pin_memory()
    qh = torch.empty(qd.shape, dtype=torch.float32).pin_memory()
    fgf.fgf_filter_host(Ih, ph, qh, 3, 540, 960, 1, 1, prm["r"], prm["eps"], prm["s"],
                        prm["sub_mode"], 0)
    assert torch.equal(qh, qd.cpu())
    # pageable host memory works too
    qh2 = torch.empty(qd.shape, dtype=torch.float32)
    fgf.fgf_filter_host(I.cpu(), p.cpu(), qh2, 3, 540, 960, 1, 1, prm["r"], prm["eps"],
                        prm["s"], prm["sub_mode"], 0)
    assert torch.equal(qh2, qd.cpu())


@pytest.mark.parametrize("B,C_I,C_p,H,W,r,s", [
    (3, 1, 1, 540, 960, 16, 4),      # H % s == 0: one 2-D copy per chunk
    (2, 1, 2, 541, 962, 8, 4),       # ragged H: one 2-D copy per plane; two p channels
    (2, 3, 1, 300, 1024, 12, 3),     # colour guidance (strip engine), odd s
    (1, 1, 1, 2050, 8192, 64, 2),    # r' = 32: K5 reading the samples in place; several chunks' worth
    (1, 1, 1, 1083, 1030, 8, 4),     # ONE gray frame: the row-band pipeline; partial last group (3 rows)
    (1, 1, 1, 1081, 2052, 16, 4),    # ... a last group of the sample row alone
    (1, 1, 1, 999, 1200, 9, 3),      # ... odd s, H a multiple of s
])
def test_host_entry_point_reads_only_sample_rows_of_p(B, C_I, C_p, H, W, r, s):
    """With nearest samples Alg. 2 reads p only at p[y s][x s]:
    fgf_filter_host copies only rows y s of p.  NaN in every other row of the host buffer
    must not reach q, which equals the device path on the clean p bit for bit; the byte count
    the library reports follows the same rule."""
    g = torch.Generator(device="cuda").manual_seed(H + W + s)
    I = torch.rand((B, C_I, H, W), device="cuda", generator=g)
    p = torch.rand((B, C_p, H, W), device="cuda", generator=g)
    qd = gpu_filter(I, p, r, 0.01, s, 0)
    ph = p.cpu()
    mask = torch.ones(H, dtype=torch.bool)
    mask[::s] = False
    ph[:, :, mask, :] = float("nan")
    Ih, ph = I.cpu().pin_memory(), ph.pin_memory()
    qh = torch.empty(qd.shape, dtype=torch.float32).pin_memory()
    fgf.fgf_filter_host(Ih, ph, qh, B, H, W, C_I, C_p, r, 0.01, s, 0, 0)
    assert torch.isfinite(qh).all()
    assert torch.equal(qh, qd.cpu())
    h = -(-H // s)
    assert fgf.fgf_filter_host_input_bytes(B, H, W, C_I, C_p, r, s, 0) == 4 * B * (C_I * H * W + C_p * h * W)
    # block means read all of p; so do s = 1, and narrow rows (< 2 KB) take the dense copy
    assert fgf.fgf_filter_host_input_bytes(B, H, W, C_I, C_p, r, s, 1) == 4 * B * (C_I + C_p) * H * W
    assert fgf.fgf_filter_host_input_bytes(B, H, W, C_I, C_p, r, 1, 0) == 4 * B * (C_I + C_p) * H * W
    assert fgf.fgf_filter_host_input_bytes(1, 64, 64, 1, 1, 8, 4, 0) == 4 * 2 * 64 * 64
    assert fgf.fgf_filter_host_input_bytes(1, 64, 64, 1, 1, 8, 4, 0, self_guided=True) == 4 * 64 * 64


@pytest.mark.parametrize("dt,B,C_I,C_p,H,W,r,s,sub", [
    ("u8", 3, 1, 1, 540, 2048, 16, 4, 0),     # 8-bit frames, sample rows of p only (2 KB rows)
    ("u8", 2, 1, 1, 301, 403, 8, 4, 0),       # odd plane sizes, narrow rows: dense copy of p
    ("f16", 2, 1, 1, 540, 1920, 16, 4, 0),
    ("bf16", 1, 3, 3, 270, 1024, 8, 2, 1),    # colour, block means: dense copy
    ("u8", 2, 3, 1, 300, 2048, 12, 3, 0),     # colour guidance, odd s
    ("u8", 1, 1, 1, 1083, 2051, 16, 4, 0),    # ONE 8-bit frame: the row-band pipeline, odd row bytes
    ("f16", 1, 1, 1, 1081, 1026, 8, 4, 0),    # ... 16-bit, a last group of the sample row alone
    ("bf16", 1, 1, 1, 720, 1280, 12, 3, 0),
])
def test_host_entry_point_reduced_precision(dt, B, C_I, C_p, H, W, r, s, sub):
    """fgf_filter_host_ex: host buffers of 8-bit codes / 16-bit floats through the same
    pipeline -- bit-identical to the device entry point on the same values."""
    tdt = {"u8": torch.uint8, "f16": torch.float16, "bf16": torch.bfloat16}[dt]
    code = {"u8": fgf.FGF_U8, "f16": fgf.FGF_F16, "bf16": fgf.FGF_BF16}[dt]
    g = torch.Generator(device="cuda").manual_seed(H + W + s)
    def mk(C):
        t = torch.rand((B, C, H, W), device="cuda", generator=g)
        return (t * 255).round().to(torch.uint8) if dt == "u8" else t.to(tdt)
    I, p = mk(C_I), mk(C_p)
    qd = fgf.filter(I, p, r, 0.01, s, sub)
    torch.cuda.synchronize()
    assert qd.dtype == tdt
    Ih, ph = I.cpu().pin_memory(), p.cpu().pin_memory()
    qh = torch.empty(qd.shape, dtype=tdt).pin_memory()
    fgf.fgf_filter_host_ex(Ih, ph, qh, B, H, W, C_I, C_p, r, 0.01, s, sub, code, 0)
    assert torch.equal(qh, qd.cpu())
    es = 1 if dt == "u8" else 2
    rows = -(-H // s) if (sub == 0 and s > 1 and W * es >= 2048) else H
    assert fgf.fgf_filter_host_input_bytes(B, H, W, C_I, C_p, r, s, sub, code) == \
        es * B * (C_I * H * W + C_p * rows * W)


def test_default_stream_entry_point():
    I, p = synth.make_batch(0, "cuda")
    q = torch.empty_like(I)
    fgf.fgf_filter(I, p, q, 1, 256, 256, 1, 1, 8, 0.01, 4, 0)
    torch.cuda.synchronize()
    assert torch.equal(q, gpu_filter(I, p, 8, 0.01, 4, 0))


def test_device_errors():
    I = torch.rand((1, 1, 64, 64), device="cuda")
    q = torch.empty_like(I)
    assert fgf.fgf_filter(I, I, I, 1, 64, 64, 1, 1, 8, 0.01, 4, 0, check=False) == fgf.FGF_ERR_ALIAS
    ws = torch.empty(16, dtype=torch.uint8, device="cuda")
    assert fgf.fgf_filter_ws(I, I, q, 1, 64, 64, 1, 1, 8, 0.01, 4, 0, ws, 16, None,
                             check=False) == fgf.FGF_ERR_NOMEM
    Ih = torch.rand((1, 1, 64, 64))
    assert fgf.fgf_filter_host(I, I, Ih, 1, 64, 64, 1, 1, 8, 0.01, 4, 0, 0,
                               check=False) == fgf.FGF_ERR_DEVICE


def test_multi_chunk_pipeline_equals_single_chunk(monkeypatch):
    """A batch larger than one pipeline slot runs as several chunks (low-res chain of chunk j
    on the library's second stream while K4 of chunk j-1 streams): same result, bit for bit,
    as one chunk; covers K13 (gray) and the strip engine (colour)."""
    monkeypatch.setenv("FGF_DEV", "1")   # honour the development knobs
    for cfg, H, W in [(1, 1080, 1920), (3, 135, 240)]:   # 6 and 2 chunks at 1 MB per slot
        I, p = synth.make_batch(cfg, "cuda", batch=6, H=H, W=W)
        prm = synth.params(cfg)
        monkeypatch.delenv("FGF_CHUNK_MB", raising=False)
        q1 = gpu_filter(I, p, **prm)
        monkeypatch.setenv("FGF_CHUNK_MB", "1")        # ~1 MB of low-res workspace per slot
        q2 = gpu_filter(I, p, **prm)
        torch.cuda.synchronize()
        assert torch.equal(q1, q2), cfg


def test_debug_sync_mode(monkeypatch):
    """FGF_DEBUG_SYNC=1 (synchronise after every launch) changes nothing in the results."""
    I, p = synth.make_batch(1, "cuda", batch=2, H=270, W=480)
    prm = synth.params(1)
    q1 = gpu_filter(I, p, **prm)
    monkeypatch.setenv("FGF_DEBUG_SYNC", "1")
    q2 = gpu_filter(I, p, **prm)
    assert torch.equal(q1, q2)


@pytest.mark.parametrize("CP", [2, 3, 4])
def test_k4_variants_agree(monkeypatch, CP):
    """The opt-in K4 variants (channel-split walker with the mbarrier ring, FGF_K4_SPLIT; the
    register-prefetch walker, FGF_NO_ASYNC) compute the same per-pixel expression in the same
    order as the default cp.async walker (as does the one-pixel-per-thread walker,
    FGF_K4_PX1), and the ungrouped colour box of a, b
    (FGF_MEAN_NOGROUP) the same sums as the grouped one: identical q, and within tolerance of
    the oracle."""
    monkeypatch.setenv("FGF_DEV", "1")   # honour the development knobs
    g = torch.Generator().manual_seed(31 + CP)
    B, H, W = 2, 203, 964                        # ragged rows, W % 4 == 0, several column blocks
    I = torch.rand((B, 3, H, W), generator=g).cuda()
    p = torch.rand((B, CP, H, W), generator=g).cuda()
    q0 = gpu_filter(I, p, 8, 0.01, 4, 1)
    for knob in ("FGF_K4_SPLIT", "FGF_NO_ASYNC", "FGF_MEAN_NOGROUP", "FGF_K4_PX1"):
        monkeypatch.setenv(knob, "1")
        q1 = gpu_filter(I, p, 8, 0.01, 4, 1)
        torch.cuda.synchronize()
        monkeypatch.delenv(knob)
        assert torch.equal(q0, q1), knob
    ref = oracle.fast_guided_filter(I[:1].cpu().numpy(), p[:1].cpu().numpy(), 8, 0.01, 4, 1)
    assert np.abs(q0[:1].double().cpu().numpy() - ref).max() <= 1e-4


@pytest.mark.parametrize("cfg,chunk_mb", [(1, None), (3, None), (1, "1")])
def test_cuda_graph_capture_and_replay(monkeypatch, cfg, chunk_mb):
    """fgf_filter_ws is capturable into a CUDA graph (small single-image calls replay without
    per-launch host overhead): the replayed graph writes the same q, bit for bit, as the eager
    call -- gray (K13 + K4), colour (K0, K1, K3, K4) and the two-stream chunk pipeline (fork /
    join through events inside the capture)."""
    monkeypatch.setenv("FGF_DEV", "1")   # honour the development knobs
    if chunk_mb:
        monkeypatch.setenv("FGF_CHUNK_MB", chunk_mb)
    else:
        monkeypatch.delenv("FGF_CHUNK_MB", raising=False)
    H, W, B = (540, 960, 4) if cfg == 1 else (270, 480, 2)
    I, p = synth.make_batch(cfg, "cuda", batch=B, H=H, W=W)
    prm = synth.params(cfg)
    CI, CP = I.shape[1], p.shape[1]
    nb = fgf.fgf_workspace_bytes(B, H, W, CI, CP, prm["r"], prm["s"])
    ws = torch.empty(nb, dtype=torch.uint8, device="cuda")
    q_ref = torch.empty((B, CP, H, W), device="cuda")
    q = torch.empty_like(q_ref)
    side = torch.cuda.Stream()
    args = (B, H, W, CI, CP, prm["r"], prm["eps"], prm["s"], prm["sub_mode"], ws, nb)
    with torch.cuda.stream(side):
        fgf.fgf_filter_ws(I, p, q_ref, *args, side)          # eager (also warms up)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=side):
        fgf.fgf_filter_ws(I, p, q, *args, side)
    q.zero_()
    g.replay()
    torch.cuda.synchronize()
    assert torch.equal(q, q_ref)


@pytest.mark.parametrize("cfg", [2, 3])
def test_colour_stats_cta_widths_agree(monkeypatch, cfg):
    """The colour statistics and box-of-a,b kernels at their narrow CTAs (default: 64 / 128
    threads) and at the plan's 256-thread width (FGF_STATS_NT256, FGF_MEAN_NT256): both within
    tolerance of the oracle, and of each other."""
    monkeypatch.setenv("FGF_DEV", "1")   # honour the development knobs
    H, W = (300, 400) if cfg == 2 else (270, 480)
    I, p = synth.make_batch(cfg, "cuda", batch=1, H=H, W=W)
    prm = synth.params(cfg)
    q128 = gpu_filter(I, p, **prm)
    monkeypatch.setenv("FGF_STATS_NT256", "1")
    monkeypatch.setenv("FGF_MEAN_NT256", "1")
    q256 = gpu_filter(I, p, **prm)
    tol = 1e-4 if prm["eps"] >= 1e-3 else 1e-3
    assert compare(I, p, q128, **prm) <= tol
    assert compare(I, p, q256, **prm) <= tol
    assert float((q128 - q256).abs().max()) <= tol


@pytest.mark.parametrize("cfg", [0, 1, 3])
def test_library_graph_cache(monkeypatch, cfg):
    """Small calls repeated with the same arguments on a non-default stream are replayed from
    the library's CUDA-graph cache (captured on the second occurrence): bit-identical q to the
    eager path (FGF_GRAPHS=0), new input VALUES are seen by the replay, the reported launch
    count is the graph's."""
    H, W, B = (256, 256, 1) if cfg == 0 else ((540, 960, 1) if cfg == 1 else (270, 480, 2))
    I, p = synth.make_batch(cfg, "cuda", batch=B, H=H, W=W)
    prm = synth.params(cfg)
    CI, CP = I.shape[1], p.shape[1]
    nb = fgf.fgf_workspace_bytes(B, H, W, CI, CP, prm["r"], prm["s"])
    ws = torch.empty(nb, dtype=torch.uint8, device="cuda")
    st = torch.cuda.Stream()
    st.wait_stream(torch.cuda.current_stream())
    args = (B, H, W, CI, CP, prm["r"], prm["eps"], prm["s"], prm["sub_mode"], ws, nb, st)
    monkeypatch.setenv("FGF_GRAPHS", "0")
    q_ref = torch.empty((B, CP, H, W), device="cuda")
    fgf.fgf_filter_ws(I, p, q_ref, *args)
    n_eager = fgf.fgf_last_launch_count()
    monkeypatch.delenv("FGF_GRAPHS")
    q = torch.empty_like(q_ref)
    for _ in range(4):                    # eager, capture + replay, replay, replay
        q.zero_()
        st.synchronize()
        fgf.fgf_filter_ws(I, p, q, *args)
        assert fgf.fgf_last_launch_count() == n_eager
        st.synchronize()
        assert torch.equal(q, q_ref)
    # new input values through the cached graph
    I2 = (I * 0.5 + 0.25).contiguous()
    I.copy_(I2)
    if cfg == 0:
        p = I
    torch.cuda.synchronize()
    fgf.fgf_filter_ws(I, p, q, *args)
    st.synchronize()
    assert compare(I, p, q, **prm) <= tol(prm["eps"])


@pytest.mark.parametrize("B,H,W,r,s,sub,eps,selfg", [
    (1, 256, 256, 8, 4, 0, 0.01, True),       # BASELINE.json config 0's geometry
    (3, 203, 301, 7, 4, 0, 0.01, False),      # ragged, several images
    (1, 251, 253, 16, 4, 1, 0.01, False),     # block mean, partial edge blocks (63 x 64)
    (2, 64, 64, 8, 1, 0, 1e-6, False),        # s = 1 (64 x 64 low-res), eps class 1e-3
    (1, 97, 370, 3, 3, 0, 0.02, False),       # odd s (33 x 124)
    (1, 5, 7, 1, 2, 0, 0.01, False),          # tiny
])
def test_tiny_single_kernel(B, H, W, r, s, sub, eps, selfg):
    """K6 (csrc/fgf_tiny.cuh): the whole filter of a small gray image (<= 4096 low-res samples,
    r' <= 8) in ONE kernel -- vs the oracle, and vs K13 + K4 on the same inputs."""
    import os
    g = torch.Generator(device="cuda").manual_seed(H + W + r + s)
    I = torch.rand((B, 1, H, W), device="cuda", generator=g)
    p = I if selfg else torch.rand((B, 1, H, W), device="cuda", generator=g)
    fgf.fgf_profile_enable(True)
    q = fgf.filter(I, p, r, eps, s, sub)
    torch.cuda.synchronize()
    prof = fgf.fgf_profile_read()
    fgf.fgf_profile_enable(False)
    assert {k: v[1] for k, v in prof.items() if v[1]} == {"tiny_fused": 1}, prof
    assert compare(I, p, q, r, eps, s, sub) <= tol(eps)
    old = {k: os.environ.get(k) for k in ("FGF_DEV", "FGF_ENGINE")}
    os.environ.update(FGF_DEV="1", FGF_ENGINE="notiny")
    try:
        q2 = fgf.filter(I, p, r, eps, s, sub)
        torch.cuda.synchronize()
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v
    assert float((q - q2).abs().max()) <= 2e-6
