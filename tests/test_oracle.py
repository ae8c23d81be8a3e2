"""Pins of the CPU oracle against what the paper and mathematics fix (CPU only).

Each test names the pin of DESIGN.md "Oracle pins" (P1-P16) and the passage it follows.
None of these compare the oracle with itself: the references are golden fixtures
(tests/golden, each cited), brute force (tests/brute.py), closed forms or identities.
"""
from __future__ import annotations

import os
from fractions import Fraction

import numpy as np
import pytest

import oracle
from tests import brute

pytestmark = pytest.mark.filterwarnings("ignore")


def load_golden(path):
    """Parse a golden fixture: '# ...' comments, then 'input H W' / 'output H W' blocks."""
    blocks = {}
    with open(path) as f:
        lines = [l.strip() for l in f if l.strip() and not l.startswith("#")]
    i = 0
    while i < len(lines):
        name, H, W = lines[i].split()
        H, W = int(H), int(W)
        rows = [[float(Fraction(t)) for t in lines[i + 1 + k].split()] for k in range(H)]
        blocks[name] = np.array(rows, np.float64).reshape(H, W)
        i += H + 1
    return blocks


# ---------------------------------------------------------------- golden fixtures (P1, P11)

def test_golden_box_impulse(golden_dir):
    g = load_golden(os.path.join(golden_dir, "box_impulse_5x5_r1.txt"))
    np.testing.assert_allclose(oracle.box_mean(g["input"], 1), g["output"], rtol=0, atol=1e-15)


def test_golden_box_clipped(golden_dir):
    g = load_golden(os.path.join(golden_dir, "box_clipped_3x3_r1.txt"))
    np.testing.assert_allclose(oracle.box_mean(g["input"], 1), g["output"], rtol=0, atol=1e-14)


def test_golden_upsample(golden_dir):
    g = load_golden(os.path.join(golden_dir, "upsample_2x2_to_4x4.txt"))
    np.testing.assert_allclose(oracle.upsample(g["input"], 4, 4), g["output"], rtol=0, atol=1e-15)


@pytest.mark.parametrize("name,mode", [("subsample_nearest_4x4_s2.txt", 0),
                                       ("subsample_block_4x4_s2.txt", 1),
                                       ("subsample_block_ragged_5x3_s2.txt", 1)])
def test_golden_subsample(golden_dir, name, mode):
    g = load_golden(os.path.join(golden_dir, name))
    np.testing.assert_allclose(oracle.subsample(g["input"], 2, mode), g["output"], rtol=0,
                               atol=1e-14)


def test_golden_radius(golden_dir):
    rows = np.loadtxt(os.path.join(golden_dir, "radius_lowres.txt"), dtype=int, comments="#")
    for r, s, rl in rows:
        assert oracle.radius_lowres(int(r), int(s)) == rl, (r, s)


def test_lowres_dims():
    # R6: ceil(dim/s)
    for D in range(1, 40):
        for s in range(1, 9):
            assert oracle.lowres_dim(D, s) == -(-D // s)


# ---------------------------------------------------------------- P1 box vs brute force

def test_box_vs_brute_force():
    rng = np.random.default_rng(1)
    for trial in range(60):
        h, w = rng.integers(1, 17, size=2)
        X = rng.random((h, w))
        for r in (1, 2, 3, 7):
            np.testing.assert_allclose(oracle.box_mean(X, r), brute.box_brute(X, r), rtol=0,
                                       atol=1e-12)


def test_box_constant_and_range():
    # S:108 constant -> constant; P13 / S:121 range preservation.
    rng = np.random.default_rng(2)
    for r in (1, 4, 40):
        c = np.full((13, 29), 0.37)
        np.testing.assert_allclose(oracle.box_mean(c, r), c, rtol=0, atol=1e-14)
        X = rng.random((31, 17))
        m = oracle.box_mean(X, r)
        assert m.min() >= X.min() - 1e-14 and m.max() <= X.max() + 1e-14


def test_box_interior_exact():
    # interior pixel = unclipped window mean.
    rng = np.random.default_rng(3)
    X = rng.random((40, 40))
    r = 5
    m = oracle.box_mean(X, r)
    for (y, x) in [(10, 10), (20, 31), (5, 5), (34, 34)]:
        assert abs(m[y, x] - X[y - r:y + r + 1, x - r:x + r + 1].mean()) < 1e-14


# ---------------------------------------------------------------- P11 resampling

def test_subsample_nearest_is_slicing():
    rng = np.random.default_rng(4)
    for (H, W, s) in [(16, 16, 4), (17, 23, 4), (9, 5, 2), (30, 31, 8), (7, 7, 1)]:
        X = rng.random((H, W))
        np.testing.assert_array_equal(oracle.subsample(X, s, 0), X[::s, ::s])


def test_subsample_block_is_reshape_mean():
    rng = np.random.default_rng(5)
    X = rng.random((24, 32))
    for s in (1, 2, 4, 8):
        ref = X.reshape(24 // s, s, 32 // s, s).mean(axis=(1, 3))
        np.testing.assert_allclose(oracle.subsample(X, s, 1), ref, rtol=0, atol=1e-14)
    Y = rng.random((19, 13))
    np.testing.assert_allclose(oracle.subsample(Y, 4, 1), brute.subsample_brute(Y, 4, 1),
                               rtol=0, atol=1e-14)


def test_upsample_properties():
    rng = np.random.default_rng(6)
    # constant -> constant, 1x1 -> fill
    np.testing.assert_allclose(oracle.upsample(np.full((5, 7), 0.25), 20, 28), 0.25, atol=1e-15)
    np.testing.assert_allclose(oracle.upsample(np.array([[0.7]]), 9, 4), 0.7, atol=1e-15)
    # s = 1 identity, bit-exact
    X = rng.random((11, 13))
    np.testing.assert_array_equal(oracle.upsample(X, 11, 13), X)
    # linearity
    A, B = rng.random((6, 9)), rng.random((6, 9))
    np.testing.assert_allclose(oracle.upsample(2 * A - 3 * B, 24, 36),
                               2 * oracle.upsample(A, 24, 36) - 3 * oracle.upsample(B, 24, 36),
                               atol=1e-13)
    # range preservation
    U = oracle.upsample(A, 24, 36)
    assert U.min() >= A.min() - 1e-15 and U.max() <= A.max() + 1e-15
    # matches the separable interpolation-matrix form, incl. ragged ratios
    for (h, w, H, W) in [(6, 9, 24, 36), (5, 3, 17, 10), (1, 4, 3, 13), (64, 64, 256, 256)]:
        M = rng.random((h, w))
        np.testing.assert_allclose(oracle.upsample(M, H, W), brute.upsample_brute(M, H, W),
                                   atol=1e-13)


def test_upsample_affine_interior():
    # A ramp M[y][x] = 0.5 + 0.25 x - 0.125 y is reproduced exactly wherever the source
    # coordinate is not clamped: value = 0.5 + 0.25 xs - 0.125 ys, xs = (X+1/2)/4 - 1/2.
    h, w, s = 8, 10, 4
    yy, xx = np.mgrid[0:h, 0:w]
    M = 0.5 + 0.25 * xx - 0.125 * yy
    U = oracle.upsample(M, h * s, w * s)
    for Y in range(2, h * s - 2):
        for X in range(2, w * s - 2):
            ys, xs = (Y + 0.5) / s - 0.5, (X + 0.5) / s - 0.5
            assert abs(U[Y, X] - (0.5 + 0.25 * xs - 0.125 * ys)) < 1e-14


# ---------------------------------------------------------------- P2/P3/P10 Eq.2-4 vs ridge

def test_guided_filter_vs_ridge_brute_force():
    """Acceptance 1 of S:463 / P2, P3, P10: Alg.1 (= FGF at s=1) equals per-window ridge
    regression + window averaging on 200 random <=16x16 images, 1 and 3 channels."""
    rng = np.random.default_rng(7)
    worst = 0.0
    for trial in range(200):
        h, w = (int(v) for v in rng.integers(2, 17, size=2))
        C = 1 if trial % 2 == 0 else 3
        r = int(rng.choice([1, 2, 3, 7]))
        eps = float(rng.choice([1e-4, 0.04]))
        I = rng.random((C, h, w)).astype(np.float32)
        p = rng.random((h, w)).astype(np.float32)
        q = oracle.guided_filter(I[None], p[None, None], r, eps)[0, 0]
        ref = brute.guided_filter_brute(I.astype(np.float64), p.astype(np.float64), r, eps)
        worst = max(worst, np.abs(q - ref).max())
    assert worst < 1e-10, worst


@pytest.mark.parametrize("C,mode", [(1, 0), (1, 1), (3, 0), (3, 1)])
def test_fgf_composition(C, mode):
    """P12 / S:250: FGF = subsample -> Alg.1 statistics at low res -> upsample -> blend,
    composed from brute-force pieces (64x64 gray, 32x40 color; s = 2, r = 4)."""
    rng = np.random.default_rng(8 + C + mode)
    H, W = (64, 64) if C == 1 else (32, 40)
    I = rng.random((C, H, W)).astype(np.float32)
    p = rng.random((H, W)).astype(np.float32)
    q = oracle.fast_guided_filter(I[None], p[None, None], 4, 0.01, 2, mode)[0, 0]
    ref = brute.fast_guided_filter_brute(I.astype(np.float64), p.astype(np.float64), 4, 0.01, 2,
                                         mode)
    assert np.abs(q - ref).max() < 1e-10


def test_fgf_ragged_composition():
    """P12 on sizes not divisible by s (partial blocks, R6) and s > r (r' clipped to 1)."""
    rng = np.random.default_rng(9)
    for (H, W, r, s, mode) in [(23, 17, 3, 4, 0), (23, 17, 3, 4, 1), (13, 30, 1, 3, 0),
                               (9, 9, 10, 2, 1)]:
        I = rng.random((H, W)).astype(np.float32)
        p = rng.random((H, W)).astype(np.float32)
        q = oracle.fast_guided_filter(I, p, r, 0.02, s, mode)[0, 0]
        ref = brute.fast_guided_filter_brute(I.astype(np.float64), p.astype(np.float64), r, 0.02,
                                             s, mode)
        assert np.abs(q - ref).max() < 1e-10, (H, W, r, s, mode)


# ---------------------------------------------------------------- identities P4-P9, P14

def _textured(rng, C, H, W):
    return rng.random((1, C, H, W)).astype(np.float32)


@pytest.mark.parametrize("C,s,mode", [(1, 1, 0), (1, 4, 0), (1, 4, 1), (3, 4, 0), (3, 2, 1)])
def test_constant_p_gives_p(C, s, mode):
    """P4: cov = 0 -> a = 0, b = c -> q = c."""
    rng = np.random.default_rng(10)
    I = _textured(rng, C, 48, 40)
    p = np.full((1, 2, 48, 40), 0.3, np.float32)
    p[:, 1] = 0.8
    q = oracle.fast_guided_filter(I, p, 8, 1e-6, s, mode)
    np.testing.assert_allclose(q[0, 0], 0.3, atol=1e-9)
    np.testing.assert_allclose(q[0, 1], 0.8, atol=1e-9)


@pytest.mark.parametrize("s", [1, 2, 4])
def test_self_guided_eps_to_zero(s):
    """P5: p = I textured, eps -> 0 -> a -> 1, b -> 0 -> q ~ I."""
    rng = np.random.default_rng(11)
    I = _textured(rng, 1, 64, 64)
    q = oracle.fast_guided_filter(I, I, 8, 1e-6, s)
    assert np.abs(q[0, 0] - I[0, 0]).max() < 1e-3


@pytest.mark.parametrize("C,s,mode", [(1, 4, 0), (1, 2, 1), (3, 4, 0)])
def test_eps_to_infinity(C, s, mode):
    """P6: eps -> inf gives a -> 0, q = upsample(f(f(p'))).  Reference built from
    brute-force subsample / box / interpolation matrices."""
    rng = np.random.default_rng(12)
    H, W, r = 40, 36, 6
    I = _textured(rng, C, H, W)
    p = rng.random((1, 1, H, W)).astype(np.float32)
    q = oracle.fast_guided_filter(I, p, r, 1e12, s, mode)[0, 0]
    rl = brute.lowres_radius(r, s)
    ps = brute.subsample_brute(p[0, 0].astype(np.float64), s, mode)
    ref = brute.upsample_brute(brute.box_brute(brute.box_brute(ps, rl), rl), H, W)
    assert np.abs(q - ref).max() < 1e-9


@pytest.mark.parametrize("C", [1, 3])
def test_shift_invariance(C):
    """P7: I + c leaves q unchanged (centred moments; b absorbs the shift)."""
    rng = np.random.default_rng(13)
    # I on a 2^-13 grid in [0, 0.5): I + 0.25 is then exact in fp32.
    I = (np.floor(_textured(rng, C, 32, 48) * 4096) / 8192).astype(np.float32)
    p = rng.random((1, 2, 32, 48)).astype(np.float32)
    q0 = oracle.fast_guided_filter(I, p, 8, 0.01, 4)
    q1 = oracle.fast_guided_filter(I + np.float32(0.25), p, 8, 0.01, 4)
    assert np.abs(q0 - q1).max() < 1e-9


@pytest.mark.parametrize("C", [1, 3])
def test_scale_invariance(C):
    """P8: c I with c^2 eps leaves q unchanged (c = 2, exact in fp32)."""
    rng = np.random.default_rng(14)
    I = _textured(rng, C, 32, 48) * 0.5
    p = rng.random((1, 1, 32, 48)).astype(np.float32)
    q0 = oracle.fast_guided_filter(I, p, 8, 0.01, 4, 1)
    q1 = oracle.fast_guided_filter(I * np.float32(2.0), p, 8, 0.04, 4, 1)
    assert np.abs(q0 - q1).max() < 1e-9


@pytest.mark.parametrize("s,mode", [(1, 0), (4, 0), (4, 1)])
def test_color_replicated_gray_equals_gray_eps_over_3(s, mode):
    """P9: with I_0 = I_1 = I_2 = g, Sherman-Morrison gives (sigma^2 11^T + eps U)^-1 1 =
    1/(3 sigma^2 + eps) 1, so sum_j a_j g = cov/(sigma^2 + eps/3) g: the color path equals
    the gray path at eps/3."""
    rng = np.random.default_rng(15)
    g = rng.random((1, 1, 40, 44)).astype(np.float32)
    p = rng.random((1, 1, 40, 44)).astype(np.float32)
    q3 = oracle.fast_guided_filter(np.repeat(g, 3, axis=1), p, 8, 0.03, s, mode)
    q1 = oracle.fast_guided_filter(g, p, 8, 0.01, s, mode)
    assert np.abs(q3 - q1).max() < 1e-9


def test_multichannel_p_independent():
    """R10: each p channel is filtered independently with the shared guidance."""
    rng = np.random.default_rng(16)
    I = _textured(rng, 3, 24, 32)
    p = rng.random((1, 3, 24, 32)).astype(np.float32)
    q = oracle.fast_guided_filter(I, p, 4, 0.01, 2, 1)
    for c in range(3):
        qc = oracle.fast_guided_filter(I, p[:, c:c + 1], 4, 0.01, 2, 1)
        np.testing.assert_array_equal(q[:, c], qc[:, 0])


def test_batch_is_independent():
    rng = np.random.default_rng(17)
    I = rng.random((3, 1, 20, 24)).astype(np.float32)
    p = rng.random((3, 1, 20, 24)).astype(np.float32)
    q = oracle.fast_guided_filter(I, p, 4, 0.01, 2)
    for b in range(3):
        np.testing.assert_array_equal(q[b], oracle.fast_guided_filter(I[b:b + 1], p[b:b + 1], 4,
                                                                      0.01, 2)[0])


def test_intermediates_consistent():
    """coefficients() + upsample_output() compose to fast_guided_filter(), and the
    mean maps are the box means of the a, b maps."""
    rng = np.random.default_rng(18)
    I = _textured(rng, 3, 33, 45)
    p = rng.random((1, 2, 33, 45)).astype(np.float32)
    mab, ab = oracle.coefficients(I, p, 8, 0.01, 4, 0, with_ab=True)
    rl = oracle.radius_lowres(8, 4)
    for c in range(2):
        for m in range(4):
            np.testing.assert_allclose(mab[0, c, m], brute.box_brute(ab[0, c, m], rl), atol=1e-12)
    q = oracle.upsample_output(I, mab, 4)
    np.testing.assert_array_equal(q, oracle.fast_guided_filter(I, p, 8, 0.01, 4, 0))


def test_finite_outputs_and_unclamped():
    """P14 and R11: finite, and q may leave [0, 1]."""
    rng = np.random.default_rng(19)
    I = (rng.random((1, 3, 64, 64)) > 0.5).astype(np.float32)   # noise-free, singular Sigma
    p = (rng.random((1, 1, 64, 64)) > 0.5).astype(np.float32)
    q = oracle.fast_guided_filter(I, p, 8, 1e-6, 4)
    assert np.isfinite(q).all()
    g = rng.random((1, 1, 64, 64)).astype(np.float32)
    q2 = oracle.fast_guided_filter(g, (g > 0.5).astype(np.float32), 2, 1e-4, 1)
    assert q2.min() < 0.0 or q2.max() > 1.0


def test_rejects_invalid():
    I = np.zeros((1, 1, 8, 8), np.float32)
    for args in [(0, 0.1, 1), (2, 0.0, 1), (2, -1.0, 1), (2, 0.1, 0), (2, 0.1, 8)]:
        with pytest.raises(ValueError):
            oracle.fast_guided_filter(I, I, *args)
    # s = 1 on a 1-pixel-high image is accepted (R7)
    J = np.random.default_rng(0).random((1, 1, 1, 9)).astype(np.float32)
    assert np.isfinite(oracle.fast_guided_filter(J, J, 2, 0.1, 1)).all()


# ---------------------------------------------------------------- application: enhancement

def test_enhance_identities():
    """gain = 1 returns the input exactly, gain = 0 returns the base layer; and the
    detail layer scales linearly with the gain."""
    rng = np.random.default_rng(31)
    I = rng.random((1, 1, 40, 52)).astype(np.float32)
    base = oracle.fast_guided_filter(I, I, 8, 0.01, 4)
    assert np.allclose(oracle.enhance(I, 1.0, 8, 0.01, 4), I.astype(np.float64), rtol=0, atol=1e-15)
    assert np.array_equal(oracle.enhance(I, 0.0, 8, 0.01, 4), base)
    e5 = oracle.enhance(I, 5.0, 8, 0.01, 4)
    assert np.allclose(e5 - base, 5.0 * (I - base), atol=1e-12)
    I3 = rng.random((1, 3, 20, 24)).astype(np.float32)
    assert np.allclose(oracle.enhance(I3, 1.0, 4, 0.01, 2), I3.astype(np.float64), rtol=0, atol=1e-15)


# ---------------------------------------------------------------- joint upsampling (R18)

@pytest.mark.parametrize("sub", [0, 1])
def test_joint_upsample_reduces_to_fgf(sub):
    """With p_low = f_sub(p, s) the joint path is Alg. 2 itself."""
    rng = np.random.default_rng(41 + sub)
    I = rng.random((1, 3, 37, 45)).astype(np.float32)
    p = rng.random((1, 2, 37, 45)).astype(np.float32)
    s, r, eps = 3, 7, 0.01
    p_low = np.stack([oracle.subsample(p[0, c], s, sub) for c in range(2)])[None]   # fp64
    q_joint = oracle.joint_upsample(I, p_low, r, eps, s, sub)
    q_fgf = oracle.fast_guided_filter(I, p, r, eps, s, sub)
    # both modes: the same fp64 I', p' on both sides (R18: steps 2-7 unchanged)
    assert np.abs(q_joint - q_fgf).max() <= 1e-12


def test_joint_upsample_constant_input():
    rng = np.random.default_rng(5)
    I = rng.random((1, 1, 40, 52)).astype(np.float32)
    p_low = np.full((1, 1, 10, 13), 0.625, np.float32)
    q = oracle.joint_upsample(I, p_low, 8, 1e-4, 4, 0)
    assert np.abs(q - 0.625).max() < 1e-9


# ---------------------------------------------------------------- luminance guidance

def test_to_grayscale_spec_examples():
    """pixel (1, 0, 0) -> 0.299; a constant (c, c, c) -> c; 1 channel -> identity."""
    px = np.array([1.0, 0.0, 0.0]).reshape(1, 3, 1, 1)
    assert abs(float(oracle.to_grayscale(px)[0, 0, 0, 0]) - 0.299) < 1e-15
    c = np.full((1, 3, 4, 5), 0.37)
    assert np.abs(oracle.to_grayscale(c) - 0.37).max() < 1e-15
    g = np.random.default_rng(0).random((2, 1, 3, 4))
    assert np.array_equal(oracle.to_grayscale(g), g)


def test_filter_f64_matches_fp32_entry_on_fp32_values():
    """fgfo_filter_f64 follows the same steps as fgfo_filter: on inputs that are exactly fp32
    values (widened exactly) the two agree to rounding of a reordered-free identical chain."""
    rng = np.random.default_rng(61)
    I = rng.random((2, 3, 29, 41)).astype(np.float32)
    p = rng.random((2, 2, 29, 41)).astype(np.float32)
    for s, sub in [(1, 0), (3, 0), (3, 1)]:
        a = oracle.fast_guided_filter(I, p, 6, 0.01, s, sub)
        b = oracle.fast_guided_filter_f64(I.astype(np.float64), p.astype(np.float64), 6, 0.01, s, sub)
        assert np.abs(a - b).max() <= 1e-14


def test_filter_f64_against_brute_force_composition():
    """On a non-fp32 (double) guidance: Alg. 2 = brute-force composition of the pinned pieces
    (subsample slicing, per-window ridge regression, interpolation matrices)."""
    from tests import brute
    rng = np.random.default_rng(62)
    H, W, r, s, eps = 22, 27, 5, 2, 0.02
    L = rng.random((1, 1, H, W)) / 3.0           # not representable in fp32
    p = rng.random((1, 1, H, W))
    q = oracle.fast_guided_filter_f64(L, p, r, eps, s, 0)
    ref = brute.fast_guided_filter_brute(L[0, 0], p[0, 0], r, eps, s, 0)
    assert np.abs(q[0, 0] - ref).max() <= 1e-12


def test_enhance_luma_identities():
    """SPEC enhance with its default shared gray guidance: gain = 1 returns
    the image, gain = 0 the base layer; an image with R = G = B = g equals the gray
    self-guided enhancement of g (its luminance is g)."""
    rng = np.random.default_rng(63)
    img = rng.random((1, 3, 33, 47)).astype(np.float32)
    assert np.abs(oracle.enhance(img, 1.0, 8, 0.01, 4, 0, guide="luma") - img).max() <= 1e-12
    base = oracle.fast_guided_filter_f64(oracle.to_grayscale(img), img, 8, 0.01, 4, 0)
    assert np.abs(oracle.enhance(img, 0.0, 8, 0.01, 4, 0, guide="luma") - base).max() <= 1e-15
    g = rng.random((1, 1, 33, 47)).astype(np.float32)
    rgb = np.repeat(g, 3, axis=1)
    e3 = oracle.enhance(rgb, 5.0, 8, 0.01, 4, 0, guide="luma")
    e1 = oracle.enhance(g, 5.0, 8, 0.01, 4, 0)
    assert np.abs(e3 - np.repeat(e1, 3, axis=1)).max() <= 1e-9
