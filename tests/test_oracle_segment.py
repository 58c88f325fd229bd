"""Pins for the oracle's NEXT-2 segmentation (Canny on the normal
image, regions between the edges).  Canny is checked against OpenCV's
cv2.Canny (a library routine with the same definition), the components
against scipy.ndimage.label.  No GPU."""
import numpy as np
import pytest

import oracle
import scenegen

cv2 = pytest.importorskip("cv2")
ndimage = pytest.importorskip("scipy.ndimage")


@pytest.mark.parametrize("seed", range(6))
def test_canny_matches_opencv(seed):
    rng = np.random.default_rng(seed)
    for _ in range(10):
        H, W = int(rng.integers(5, 80)), int(rng.integers(5, 80))
        C = int(rng.choice([1, 3]))
        kind = int(rng.integers(0, 3))
        if kind == 0:
            img = rng.integers(0, 256, (H, W, C)).astype(np.uint8)
        elif kind == 1:
            img = np.zeros((H, W, C), np.uint8)
            img[:, W // 2:] = 200
            img[H // 3:, : W // 3] = 90
        else:
            y, x = np.mgrid[0:H, 0:W]
            img = np.repeat(((np.sin(x / 3.0) + np.cos(y / 4.0)) * 60 + 128).astype(np.uint8)[..., None], C, 2)
        img = np.ascontiguousarray(img[..., 0] if C == 1 else img)
        lo, hi = float(rng.choice([10, 30, 50])), float(rng.choice([60, 90, 150]))
        assert np.array_equal(oracle.canny_u8(img, lo, hi), cv2.Canny(img, lo, hi, L2gradient=True))


def test_normals_to_u8_and_canny_on_a_normal_image():
    fr = scenegen.make_config("C2")
    n = oracle.normals(fr["depth"].numpy(), fr["K"]).astype(np.float32)
    u8 = oracle.normals_to_u8(n)
    want = np.clip(np.rint((n.transpose(1, 2, 0) + np.float32(1)) * np.float32(127.5)), 0, 255).astype(np.uint8)
    assert np.array_equal(u8, want)
    assert np.array_equal(oracle.canny_u8(u8, 30, 90), cv2.Canny(u8, 30, 90, L2gradient=True))


def test_uniform_and_step_normal_images():
    # uniform normal image -> no edges, one region (the whole image)
    H, W = 40, 50
    n = np.zeros((3, H, W), np.float32)
    n[2] = -1
    lab, nr, edges = oracle.segment_regions(n, 30, 90, 10)
    assert nr == 1 and edges.sum() == 0 and np.all(lab == 0)
    # two halves 90 deg apart -> one vertical edge line (before dilation)
    n2 = n.copy()
    n2[:, :, 25:] = np.array([1, 0, 0], np.float32)[:, None, None]
    e = oracle.canny_u8(oracle.normals_to_u8(n2), 30, 90)
    cols = np.unique(np.nonzero(e)[1])
    assert len(cols) == 1 and e[:, cols[0]].all()
    lab, nr, edges = oracle.segment_regions(n2, 30, 90, 10)
    assert nr == 2 and set(np.unique(lab)) == {-1, 0, 1}
    # an invalid-depth hole (zero normal) -> edge
    n3 = n.copy()
    n3[:, 10:14, 10:14] = 0
    lab, nr, edges = oracle.segment_regions(n3, 30, 90, 10)
    assert edges[10:14, 10:14].all() and np.all(lab[9:15, 9:15] == -1)


def test_regions_match_scipy_components():
    fr = scenegen.make_config("C2", noise=True)
    d = oracle.adf(fr["depth"].numpy(), 0.15, 0.03, 20)
    n = oracle.normals(d, fr["K"]).astype(np.float32)
    lab, nr, edges = oracle.segment_regions(n, 30, 90, 300)
    # the dilated edge mask = 3x3 dilation of (Canny | invalid)
    e0 = (oracle.canny_u8(oracle.normals_to_u8(n), 30, 90) > 0) | np.all(n == 0, axis=0)
    assert np.array_equal(edges.astype(bool), ndimage.binary_dilation(e0, structure=np.ones((3, 3)), border_value=0))
    comp, ncomp = ndimage.label(~edges.astype(bool), structure=[[0, 1, 0], [1, 1, 1], [0, 1, 0]])
    sizes = ndimage.sum_labels(np.ones_like(comp), comp, index=np.arange(1, ncomp + 1)).astype(int)
    big = [c + 1 for c in range(ncomp) if sizes[c] >= 300]
    assert nr == len(big) and nr >= 4
    # each region is exactly one scipy component; ordered by size desc
    prev = None
    for r in range(nr):
        m = lab == r
        cs = np.unique(comp[m])
        assert len(cs) == 1 and cs[0] in big and m.sum() == sizes[cs[0] - 1]
        if prev is not None:
            assert m.sum() <= prev
        prev = m.sum()
    assert np.all(lab[~np.isin(comp, big)] == -1)


def test_stair_treads_become_regions():
    # noise-free staircase: every region lies on a single ground-truth tread
    fr = scenegen.make_config("C2", noise=False)
    n = oracle.normals(fr["depth"].numpy(), fr["K"]).astype(np.float32)
    lab, nr, _ = oracle.segment_regions(n, 30, 90, 300)
    face = fr["face"].numpy()
    assert nr >= 4
    for r in range(nr):
        assert len(np.unique(face[lab == r])) == 1


def test_normals_to_u8_fixed_values_channel_order_and_ties():
    """Pins orc_normals_to_u8 (NEXT-2 input) to SPEC S:197's formula
    round((n + 1) / 2 * 255) by hand-computed values, not a restatement.
    Reading (Q26): `round` is round-half-to-even (Python 3's
    round, C's rint); in f32, (n+1)/2*255 and (n+1)*127.5 are the same
    single rounding of the same real number."""
    H, W = 1, 5
    n = np.zeros((3, H, W), np.float32)
    n[0, 0] = [-1.0, -0.5, 0.0, 0.5, 1.0]          # x -> R
    n[1, 0] = [1.0, 0.5, 0.0, -0.5, -1.0]          # y -> G
    n[2, 0] = [0.0, 0.0, 0.0, 0.0, 0.0]            # z -> B: 127.5, a tie
    u8 = oracle.normals_to_u8(n)
    assert u8.shape == (H, W, 3)
    # -1 -> 0; -0.5 -> 63.75 -> 64; 0 -> 127.5 -> 128 (tie to even); 0.5 -> 191.25 -> 191; 1 -> 255
    assert u8[0, :, 0].tolist() == [0, 64, 128, 191, 255]
    assert u8[0, :, 1].tolist() == [255, 191, 128, 64, 0]
    assert u8[0, :, 2].tolist() == [128] * 5
    # exact ties k + 1/2 (f32 inputs whose f32 product lands on the tie): k even
    # rounds down, k odd rounds up (half-away-from-zero would give k + 1 for both)
    for k in (100, 101):
        target = np.float32(k + 0.5)
        v = np.float32(k + 0.5) / np.float32(127.5) - np.float32(1)
        cand = (np.arange(-4096, 4096, dtype=np.int64) + int(v.view(np.uint32))).astype(np.uint32).view(np.float32)
        hit = cand[(cand + np.float32(1)) * np.float32(127.5) == target]
        assert hit.size, f"no f32 input hits the tie {k}.5"
        t = np.zeros((3, 1, hit.size), np.float32)
        t[0, 0] = hit
        got = oracle.normals_to_u8(t)[0, :, 0]
        assert np.all(got == (k if k % 2 == 0 else k + 1)), (k, got)
