"""Pins for the paper-literal variants: Eq. 1 as the
4-flux Perona-Malik scheme and Eq. 2 taken literally.
No GPU."""
import math
import os

import numpy as np

import oracle
import scenegen

DIV = oracle.ADF_DIVERGENCE


def _golden(golden_dir, tag):
    with open(os.path.join(golden_dir, "spec_worked_examples.txt")) as f:
        return [ln.split()[1:] for ln in f if ln.startswith(tag + " ")]


def test_divergence_1d_profile(golden_dir):
    (row,) = _golden(golden_dir, "adf1d_div")
    lam, k = float(row[0]), float(row[1]) / 1000.0
    arrow = row.index("->")
    prof = np.array([float(x) for x in row[2:arrow]]) / 1000.0
    want = np.array([float(x) for x in row[arrow + 1:]])
    out = oracle.adf(prof.astype(np.float32)[None, :], lam, k, 1, scheme=DIV)[0].astype(np.float64) * 1000
    assert np.allclose(out, want, atol=1e-4 + 1e-6)


def test_divergence_impulse_closed_form():
    # one step on base + delta: every edge of p carries flux
    # lambda exp(-(delta/k)^2) delta; p loses four of them, each neighbour gains one
    base, delta, lam, kap = 1.0, 0.02, 0.15, 0.03
    d = np.full((9, 9), base, np.float32)
    d[4, 4] = base + delta
    dd = float(np.float32(base + delta)) - base
    flux = lam * math.exp(-(dd / kap) ** 2) * dd
    out = oracle.adf(d, lam, kap, 1, scheme=DIV).astype(np.float64)
    assert abs(out[4, 4] - (base + dd - 4 * flux)) < 1e-7
    for (v, u) in [(3, 4), (5, 4), (4, 3), (4, 5)]:
        assert abs(out[v, u] - (base + flux)) < 1e-7
    assert out[3, 3] == base and out[2, 4] == base


def test_divergence_conserves_mass_with_holes_and_borders():
    # fluxes are antisymmetric and zero across borders / holes: the sum of
    # valid depth is invariant (here to f32 output rounding)
    rng = np.random.default_rng(5)
    d = (1.0 + 0.02 * rng.standard_normal((40, 50))).astype(np.float32)
    d[rng.random(d.shape) < 0.05] = 0.0
    out = oracle.adf(d, 0.2, 0.03, 15, scheme=DIV)
    v = d > 0
    assert abs(out[v].astype(np.float64).sum() - d[v].astype(np.float64).sum()) < 2e-4
    # Alg. 1 as printed is not conservative on the same input
    out1 = oracle.adf(d, 0.2, 0.03, 15)
    assert abs(out1[v].astype(np.float64).sum() - d[v].astype(np.float64).sum()) > 1e-3


def test_divergence_fixed_points():
    c = np.full((10, 12), 2.5, np.float32)
    assert oracle.adf(c, 0.25, 0.05, 20, scheme=DIV).tobytes() == c.tobytes()
    # dyadic ramp: interior fluxes cancel to first order but c(d) differs
    # for d = +a and -a only by sign -> interior exactly unchanged
    v, u = np.mgrid[0:8, 0:10]
    r = (1 + u / 64 + v / 32).astype(np.float32)
    out = oracle.adf(r, 0.2, 0.05, 1, scheme=DIV)
    assert np.array_equal(out[1:-1, 1:-1], r[1:-1, 1:-1])


def test_printed_normals_constant_image(golden_dir):
    (row,) = _golden(golden_dir, "normals_printed")
    fx, fy, cx, cy = (float(x) for x in row[0:4])
    want = np.array([float(x) for x in row[5:8]])
    n = oracle.normals(np.full((12, 16), 1.0, np.float32), scenegen.Intrinsics(fx, fy, cx, cy),
                       mode=oracle.NORMALS_AS_PRINTED)
    assert np.allclose(n[:, 6, 8], want, atol=5e-4)
    assert np.allclose(n.reshape(3, -1), n[:, 6, 8][:, None])       # constant everywhere


def test_printed_normals_follow_eq2_on_a_ramp():
    # Gx = a, Gy = b exactly on a ramp -> n ∝ -((a - cx)/fx, (b - cy)/fy, 1)
    K = scenegen.intrinsics_for(64, 48)
    v, u = np.mgrid[0:48, 0:64]
    a, b = 0.5, -0.25
    D = (3.0 + a * u + b * v).astype(np.float64)
    n = oracle.normals_f64(D, K, mode=oracle.NORMALS_AS_PRINTED)[:, 20, 30]
    m = -np.array([(a - K.cx) / K.fx, (b - K.cy) / K.fy, 1.0])
    assert np.allclose(n, m / np.linalg.norm(m), atol=1e-12)
