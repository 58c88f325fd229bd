"""Pins for the oracle's Algorithm 1 ℓ9-13 (Sobel + normal), Eq. 2
 read geometrically (Q7).  No GPU."""
import numpy as np

import oracle
import scenegen


def _angle(a, b):
    """atan2(|a x b|, a.b) in float64 (robust near 0, unlike arccos)."""
    c = np.cross(a, b, axis=0)
    return np.arctan2(np.linalg.norm(c, axis=0), (a * b).sum(0))


def test_constant_depth_gives_optical_axis_exactly():
    # P8: fronto-parallel plane -> Gx = Gy = 0 -> m = (0, 0, -Z) -> (0, 0, -1) exactly
    K = scenegen.intrinsics_for(40, 30)
    n = oracle.normals(np.full((30, 40), 1.7, np.float32), K)
    assert np.all(n[0] == 0) and np.all(n[1] == 0) and np.all(n[2] == -1)


def test_sobel_on_ramp_is_exact():
    # P8 / S:170-172: Sobel/8 of a*u + b*v is (a, b) in the interior, and
    # (a/2, ...) on a clamped border column
    H, W = 9, 11
    v, u = np.mgrid[0:H, 0:W].astype(np.float64)
    g = oracle.sobel_f64(3 * u + 4 * v)
    assert np.all(g[0, 1:-1, 1:-1] == 3) and np.all(g[1, 1:-1, 1:-1] == 4)
    assert np.all(g[0, 1:-1, 0] == 1.5) and np.all(g[1, 0, 1:-1] == 2)
    assert np.all(oracle.sobel_f64(np.full((5, 6), 2.5)) == 0)


def test_tilted_plane_gives_true_normal():
    # P8 / SURVEY A.2: on an analytic plane the geometric normal from Sobel(Z)
    # is exact up to the Sobel truncation of the (hyperbolic) depth: <= 3e-6
    # rad for the survey's 30-degree plane at 640x480 and < 1.5e-5 rad for
    # steeper planes out to 4 m; any sign / axis / scale mistake is ~1e-1 rad.
    W, H = 640, 480
    K = scenegen.intrinsics_for(W, H)
    for tilt, az, tol in [(30, 35, 3e-6), (30, 0, 3e-6), (50, -120, 1.5e-5), (10, 200, 1e-7), (40, 90, 6e-6)]:
        depth, face, planes = scenegen.ramp(W, H, K, tilt_deg=tilt, azim_deg=az)
        n_true = np.array(planes[0][0])
        D = depth.numpy()
        N = oracle.normals_f64(D, K)
        ok = (np.abs(N).sum(0) > 0) & (D < 4.0)
        ok[0] = ok[-1] = False
        ok[:, 0] = ok[:, -1] = False
        assert ok.mean() > 0.75
        ang = _angle(N[:, ok], n_true[:, None])
        assert ang.max() < tol, (tilt, az, ang.max())
        # f32-rounded depth (the ABI's input type): SURVEY A.2 ~2.2e-5 rad
        N32 = oracle.normals(D.astype(np.float32), K)
        ang32 = _angle(N32[:, ok], n_true[:, None])
        assert ang32.max() < 1e-4


def test_normals_face_camera_and_are_unit():
    # Q9: m . P(u, v) = -Z^2 < 0, so every valid normal faces the camera
    fr = scenegen.make_config("C2")
    K = fr["K"]
    D = fr["depth"].numpy()
    N = oracle.normals(D, K)
    H, W = D.shape
    v, u = np.mgrid[0:H, 0:W]
    P = np.stack([(u - K.cx) / K.fx * D, (v - K.cy) / K.fy * D, D])
    ok = np.abs(N).sum(0) > 0
    assert ok.mean() > 0.99
    assert np.all((N * P).sum(0)[ok] < 0)
    assert np.abs(np.linalg.norm(N[:, ok], axis=0) - 1).max() < 1e-12


def test_invalid_window_mask():
    # Q9 / S:156: (0,0,0) iff any pixel of the clamped 3x3 window is invalid
    K = scenegen.intrinsics_for(20, 16)
    D = np.full((16, 20), 1.0, np.float32)
    D[5, 7] = 0.0
    D[0, 19] = np.nan
    N = oracle.normals(D, K)
    zero = np.all(N == 0, axis=0)
    want = np.zeros_like(zero)
    want[4:7, 6:9] = True
    want[0:2, 18:20] = True
    assert np.array_equal(zero, want)


def test_tilt_sign_and_axes():
    # a plane tilted toward +x (depth grows with u) must have n_x > 0 ...
    # i.e. the normal of Z = z0 + s u (s > 0) leans to +x before facing -z
    K = scenegen.intrinsics_for(64, 48)
    v, u = np.mgrid[0:48, 0:64]
    D = (2.0 + 0.01 * (u - K.cx)).astype(np.float64)
    N = oracle.normals_f64(D, K)[:, 24, 32]
    assert N[0] > 0 and abs(N[1]) < 1e-12 and N[2] < 0
    D2 = (2.0 + 0.01 * (v - K.cy)).astype(np.float64)
    N2 = oracle.normals_f64(D2, K)[:, 24, 32]
    assert N2[1] > 0 and abs(N2[0]) < 1e-12 and N2[2] < 0
    # exact: at the principal point m = (fx Gx, fy Gy, -Z)
    Dc = 2.0 + 0.01 * (u - 31.0)
    Nc = oracle.normals_f64(Dc, K)[:, 24, 31]
    m = np.array([K.fx * 0.01, 0.0, -(2.0 + (31 - K.cx) * 0.01)])
    assert np.allclose(Nc, m / np.linalg.norm(m), atol=1e-14)
