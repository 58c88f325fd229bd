"""Pins for the oracle's Algorithm 1 ℓ1-8 (anisotropic diffusion).

Each test checks the oracle against something other than itself: a closed
form derived from Alg. 1, an invariant of the scheme, or a worked example
(tests/golden/spec_worked_examples.txt).  No GPU.
"""
import math
import os

import numpy as np
import pytest

import oracle
import scenegen

LAM, KAP = 0.15, 0.03


def test_zero_iterations_is_identity():
    # S:119 "N=0 is the identity"; Alg. 1 ℓ1 I_smooth <- I
    rng = np.random.default_rng(0)
    d = (1 + rng.random((17, 23))).astype(np.float32)
    d[3, 4] = 0.0
    d[5, 6] = np.nan
    out = oracle.adf(d, LAM, KAP, 0)
    assert out.tobytes() == d.tobytes()


@pytest.mark.parametrize("iters", [1, 7, 50])
def test_constant_image_is_bitwise_fixed_point(iters):
    # P4: grad = 0 and lap = 0 everywhere, including borders (zero flux, Q4)
    d = np.full((16, 21), 1.2345, np.float32)
    out = oracle.adf(d, LAM, KAP, iters)
    assert out.tobytes() == d.tobytes()


def test_holes_are_zero_flux_and_never_change():
    # Q4: an invalid neighbour takes the centre value; invalid pixels keep
    # their bits (0, negative, NaN, inf)
    d = np.full((12, 12), 2.0, np.float32)
    d[2, 3], d[5, 5], d[7, 1], d[0, 0], d[11, 6] = 0.0, np.nan, -1.0, np.inf, -0.0
    out = oracle.adf(d, LAM, KAP, 5)
    assert out.tobytes() == d.tobytes()


def test_impulse_closed_form():
    # P5: one Jacobi step on base + delta at p: p -> base + delta (1 - 4 lam)
    # (its gradient is 0, so c = 1); each 4-neighbour q -> base + lam
    # exp(-(delta/2)^2 / k^2) delta (gradient delta/2 at q, lap = delta);
    # every other pixel unchanged.  Also pins Jacobi (not in-place): all
    # four neighbours must agree.
    base, delta = 1.0, 0.02
    d = np.full((9, 9), base, np.float32)
    d[4, 4] = base + delta
    out = oracle.adf(d, LAM, KAP, 1).astype(np.float64)
    dd = float(np.float32(base + delta)) - base            # the impulse as stored in f32
    centre = base + dd * (1 - 4 * LAM)
    nb = base + LAM * math.exp(-(dd / 2) ** 2 / KAP ** 2) * dd
    assert abs(out[4, 4] - centre) < 1e-7
    for (v, u) in [(3, 4), (5, 4), (4, 3), (4, 5)]:
        assert abs(out[v, u] - nb) < 1e-7, (v, u, out[v, u], nb)
    mask = np.ones_like(out, bool)
    mask[4, 4] = mask[3, 4] = mask[5, 4] = mask[4, 3] = mask[4, 5] = False
    assert np.all(out[mask] == base)
    # numbers quoted in SURVEY A.3 for this case
    assert abs(out[4, 4] - 1.008) < 1e-7 and abs(out[4, 5] - 1.0026845) < 1e-7


def test_linear_ramp_interior_and_border_closed_form():
    # Interior of a dyadic ramp I = 1 + a u + b v has lap = 0 exactly -> unchanged.
    # Left border (u = 0, 0 < v < H-1): W takes the centre value (Q4), so
    # gx = a/2, gy = b, lap = a; top-left corner: gx = a/2, gy = b/2, lap = a + b.
    a, b, kap, lam = 1 / 64, 1 / 32, 0.05, 0.2
    H, W = 8, 10
    v, u = np.mgrid[0:H, 0:W]
    d = (1 + a * u + b * v).astype(np.float32)
    out = oracle.adf(d, lam, kap, 1).astype(np.float64)
    assert np.array_equal(out[1:-1, 1:-1], d[1:-1, 1:-1])
    for vv in range(1, H - 1):
        want = d[vv, 0] + lam * math.exp(-((a / 2) ** 2 + b ** 2) / kap ** 2) * a
        assert abs(out[vv, 0] - want) < 2e-7
    want = d[0, 0] + lam * math.exp(-((a / 2) ** 2 + (b / 2) ** 2) / kap ** 2) * (a + b)
    assert abs(out[0, 0] - want) < 2e-7
    # right border: E takes the centre value: gx = a/2, lap = -a
    want = d[3, W - 1] + lam * math.exp(-((a / 2) ** 2 + b ** 2) / kap ** 2) * (-a)
    assert abs(out[3, W - 1] - want) < 2e-7


def _golden(golden_dir, tag):
    with open(os.path.join(golden_dir, "spec_worked_examples.txt")) as f:
        return [ln.split()[1:] for ln in f if ln.startswith(tag + " ")]


def test_spec_1d_profile(golden_dir):
    # S:111 worked example, Alg. 1 as printed (SURVEY A.3 values), 3 decimals
    (row,) = _golden(golden_dir, "adf1d")
    lam, k = float(row[0]), float(row[1]) / 1000.0
    arrow = row.index("->")
    prof = np.array([float(x) for x in row[2:arrow]]) / 1000.0
    want = np.array([float(x) for x in row[arrow + 1:]])
    img = np.tile(prof.astype(np.float32), (1, 1))          # a 1-row image: N/S out of image
    out = oracle.adf(img, lam, k, 1)[0].astype(np.float64) * 1000.0
    assert np.allclose(out, want, atol=1e-3 + 1e-6)
    # SPEC S:111 also claims "row sum preserved"; false for Alg. 1 as printed
    # (c_p lap is not conservative): the sum changes by about -0.00999 mm.
    assert abs((out.sum() - prof.sum() * 1000) - (-0.009988)) < 1e-3


def test_max_principle_and_noise_reduction():
    # S:126 max principle (a convex combination for lam <= 1/4); with
    # sigma = 5 mm noise on a plane, N = 10 reduces the residual by >= 40 %
    rng = np.random.default_rng(11)
    d = (1.5 + 0.005 * rng.standard_normal((64, 64))).astype(np.float32)
    out = oracle.adf(d, LAM, KAP, 10)
    assert out.min() >= d.min() and out.max() <= d.max()
    inner = (slice(2, -2), slice(2, -2))
    r0 = np.abs(d.astype(np.float64) - 1.5)[inner].mean()
    r1 = np.abs(out.astype(np.float64) - 1.5)[inner].mean()
    assert r1 < 0.6 * r0, (r0, r1)


def test_edge_preservation():
    # step 0.5 -> 2.0 m with k = 0.01 m moves by < 1 mm
    d = np.full((10, 20), 0.5, np.float32)
    d[:, 10:] = 2.0
    out = oracle.adf(d, 0.2, 0.01, 10)
    assert np.abs(out - d).max() < 1e-3


def test_symmetry_flips_and_transpose():
    # Alg. 1 is isotropic on the 5-point stencil: ADF commutes with flips
    # and the transpose (rounding-order differences only)
    rng = np.random.default_rng(3)
    d = (1 + 0.05 * rng.random((13, 17))).astype(np.float32)
    d[4, 6] = 0
    ref = oracle.adf(d, LAM, KAP, 6)
    assert np.allclose(oracle.adf(d[::-1], LAM, KAP, 6)[::-1], ref, atol=3e-7, rtol=0)
    assert np.allclose(oracle.adf(d[:, ::-1], LAM, KAP, 6)[:, ::-1], ref, atol=3e-7, rtol=0)
    assert np.allclose(oracle.adf(np.ascontiguousarray(d.T), LAM, KAP, 6).T, ref, atol=3e-7, rtol=0)


def test_composition():
    # N1 + N2 = N (the oracle rounds to f32 at each call boundary)
    fr = scenegen.make_config("C1n")
    d = fr["depth"].numpy()
    a = oracle.adf(oracle.adf(d, LAM, KAP, 4), LAM, KAP, 6)
    b = oracle.adf(d, LAM, KAP, 10)
    assert np.abs(a - b).max() < 1e-6
