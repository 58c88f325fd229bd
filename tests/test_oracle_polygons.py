"""Pins for the oracle's NEXT-3 polygon glue (S:236-251,
S:324-332): contour tracing against OpenCV's border following, Douglas-Peucker
against its contract and SPEC's examples, rasterisation against closed forms
and the partition property of its half-open rule, vertex lifting against the
plane and the reprojection.  No GPU."""
import math

import numpy as np
import pytest

import oracle
import scenegen

cv2 = pytest.importorskip("cv2")


def _canon(seq):
    seq = [tuple(int(v) for v in p) for p in seq]
    i = seq.index(min(seq, key=lambda p: (p[1], p[0])))
    return seq[i:] + seq[:i]


def _blobs(rng, H=60, W=80):
    m = np.zeros((H, W), np.uint8)
    for _ in range(int(rng.integers(1, 4))):
        cv2.ellipse(m, (int(rng.integers(10, W - 10)), int(rng.integers(10, H - 10))),
                    (int(rng.integers(2, 20)), int(rng.integers(2, 15))), float(rng.uniform(0, 180)), 0, 360, 1, -1)
    _, cc = cv2.connectedComponents(m, connectivity=8)
    return np.where(cc == 1, 0, -1).astype(np.int32)


@pytest.mark.parametrize("seed", range(4))
def test_trace_equals_opencv_border_following(seed):
    # Q35 traces clockwise on screen; cv2.findContours (Suzuki-Abe, outer
    # border, CHAIN_APPROX_NONE) gives the same pixels counter-clockwise
    rng = np.random.default_rng(seed)
    for _ in range(60):
        lab = _blobs(rng)
        if (lab == 0).sum() == 0:
            continue
        ours = oracle.trace_contour(lab, 0)
        cs, _ = cv2.findContours((lab == 0).astype(np.uint8), cv2.RETR_EXTERNAL, cv2.CHAIN_APPROX_NONE)
        assert _canon(ours) == _canon(cs[0].reshape(-1, 2)[::-1])


def test_trace_on_segmented_stair_regions():
    fr = scenegen.make_config("C2", noise=False)
    n = oracle.normals(fr["depth"].numpy(), fr["K"]).astype(np.float32)
    lab, nr, _ = oracle.segment_regions(n, 30, 90, 300)
    assert nr >= 4
    for r in range(nr):
        c = oracle.trace_contour(lab, r)
        # closed 8-connected walk through region pixels, starting at the
        # region's first pixel in raster order
        d = np.abs(np.diff(np.vstack([c, c[:1]]), axis=0))
        assert d.max() <= 1 and (d.sum(1) > 0).all()
        assert (lab[c[:, 1], c[:, 0]] == r).all()
        ys, xs = np.nonzero(lab == r)
        assert (c[0, 0], c[0, 1]) == (xs[0], ys[0])
        # the region component containing the start: its outer border equals OpenCV's
        _, cc = cv2.connectedComponents((lab == r).astype(np.uint8), connectivity=8)
        comp = (cc == cc[c[0, 1], c[0, 0]]).astype(np.uint8)
        cs, _ = cv2.findContours(comp, cv2.RETR_EXTERNAL, cv2.CHAIN_APPROX_NONE)
        assert _canon(c) == _canon(cs[0].reshape(-1, 2)[::-1])


def test_trace_degenerate():
    lab = -np.ones((5, 6), np.int32)
    assert len(oracle.trace_contour(lab, 0)) == 0
    lab[2, 3] = 0
    assert oracle.trace_contour(lab, 0).tolist() == [[3, 2]]
    lab[2, 4] = 0                                  # two pixels: there and back
    assert oracle.trace_contour(lab, 0).tolist() == [[3, 2], [4, 2]]
    full = np.zeros((4, 5), np.int32)              # region touching every border
    c = oracle.trace_contour(full, 0)
    assert len(c) == 2 * (4 + 5) - 4


def _line_dist(p, a, b):
    a, b, p = np.asarray(a, float), np.asarray(b, float), np.asarray(p, float)
    d = b - a
    if not d.any():
        return float(np.hypot(*(p - a)))
    return abs(d[0] * (p - a)[1] - d[1] * (p - a)[0]) / math.hypot(*d)


def test_dp_rectangle_and_circle_spec_examples():
    lab = -np.ones((40, 50), np.int32)
    lab[5:30, 8:41] = 0
    c = oracle.trace_contour(lab, 0)
    assert _canon(oracle.simplify_dp(c, 2.0)) == _canon([[8, 5], [40, 5], [40, 29], [8, 29]])
    yy, xx = np.mgrid[0:130, 0:130]
    lab = np.where((xx - 64) ** 2 + (yy - 64) ** 2 <= 50 ** 2, 0, -1).astype(np.int32)
    c = oracle.trace_contour(lab, 0)
    s = oracle.simplify_dp(c, 1.0)
    assert len(s) < 40


@pytest.mark.parametrize("eps", [0.5, 1.0, 3.0, 7.25])
def test_dp_contract(eps):
    # kept vertices are contour points in order, both anchors kept, and every
    # dropped point lies within eps of the line of the segment that covers it
    rng = np.random.default_rng(int(eps * 4))
    for _ in range(40):
        lab = _blobs(rng)
        c = oracle.trace_contour(lab, 0)
        if len(c) < 3:
            continue
        s, idx = oracle.simplify_dp(c, eps, return_index=True)
        idx = idx.tolist()
        assert np.array_equal(s, c[idx]) and idx[0] == 0 and idx == sorted(idx)
        far = int(np.argmax(((c - c[0]) ** 2).sum(1)))
        assert far in idx
        ring = idx + [len(c)]
        for a, b in zip(ring[:-1], ring[1:]):
            pa, pb = c[a], c[b % len(c)]
            for k in range(a + 1, b):
                assert _line_dist(c[k], pa, pb) <= eps + 1e-9


def test_rasterize_closed_forms_and_partition():
    W, H = 40, 30
    rect = [[5, 4], [25, 4], [25, 20], [5, 20]]
    lab = oracle.rasterize_polygons([rect], W, H)
    want = np.full((H, W), -1, np.int32)
    want[4:20, 5:25] = 0                           # half-open: x in [5, 25), y in [4, 20)
    assert np.array_equal(lab, want)
    # a rectangle cut along its diagonal: the two triangles partition it
    t1 = [[5, 4], [25, 4], [25, 20]]
    t2 = [[5, 4], [25, 20], [5, 20]]
    a = oracle.rasterize_polygons([t1], W, H) == 0
    b = oracle.rasterize_polygons([t2], W, H) == 0
    assert not (a & b).any() and np.array_equal(a | b, want == 0)
    # orientation does not matter; overlapping polygons -> lowest index wins
    assert np.array_equal(oracle.rasterize_polygons([rect[::-1]], W, H), want)
    lab2 = oracle.rasterize_polygons([[[0, 0], [10, 0], [10, 10], [0, 10]], rect], W, H)
    assert (lab2[4:10, 5:10] == 0).all() and (lab2[12:20, 12:25] == 1).all()
    # a random fan of triangles around a centre partitions its convex hull
    rng = np.random.default_rng(2)
    ang = np.sort(rng.uniform(0, 2 * np.pi, 9))
    pts = np.stack([20 + np.round(12 * np.cos(ang)), 15 + np.round(12 * np.sin(ang))], 1).astype(np.int32)
    fan = [[[20, 15], pts[i].tolist(), pts[(i + 1) % 9].tolist()] for i in range(9)]
    counts = sum((oracle.rasterize_polygons([t], W, H) == 0).astype(int) for t in fan)
    whole = oracle.rasterize_polygons([pts.tolist()], W, H) == 0
    assert counts.max() <= 1 and np.array_equal(counts == 1, whole)


def test_lift_vertices_on_plane_and_reprojection():
    K = scenegen.intrinsics_for(640, 480)
    rng = np.random.default_rng(5)
    for _ in range(20):
        n = rng.normal(size=3)
        n[2] = -abs(n[2]) - 0.5
        n /= np.linalg.norm(n)
        d = float(rng.uniform(0.5, 3.0))
        uv = rng.integers(0, [640, 480], size=(50, 2)).astype(np.int32)
        X = oracle.lift_vertices(uv, [*n, d], K)
        ok = np.isfinite(X).all(1)
        assert ok.any()
        assert np.abs(X[ok] @ n + d).max() < 1e-12
        assert np.allclose(X[ok, 0] / X[ok, 2] * K.fx + K.cx, uv[ok, 0], atol=1e-9)
        assert np.allclose(X[ok, 1] / X[ok, 2] * K.fy + K.cy, uv[ok, 1], atol=1e-9)
        assert (X[ok, 2] > 0).all()
