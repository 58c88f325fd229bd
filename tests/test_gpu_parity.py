"""GPU parity: the CUDA path (through the C ABI) against the oracle, element
by element, on the same seeded inputs (DESIGN.md §6 test matrix).

Tolerances (north_star / DESIGN.md §6): ADF depth |d| <= 1e-4 m on valid
pixels, invalid pixels bitwise; normals angle <= 1e-3 rad with the invalid
mask bitwise; RANSAC per-hypothesis counts, selected index, n_points and
status bit-exact; refit n, d, centroid within 1e-5."""
import math

import numpy as np
import pytest
import torch

import oracle
import scenegen

pytestmark = pytest.mark.gpu

ADF_TOL = 1e-4
ANG_TOL = 1e-3
REFIT_TOL = 1e-5


@pytest.fixture(scope="module")
def pm():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2411_01919_b200 as pm
    return pm


DEV = "cuda"


def _angle(a, b):
    c = np.cross(a, b, axis=0)
    return np.arctan2(np.linalg.norm(c, axis=0), (a * b).sum(0))


def _check_normals(n_gpu, n_ref, exclude=None):
    n_gpu = n_gpu.astype(np.float64)
    if exclude is not None:   # pixels outside the f32 representable range of |m|^2
        n_gpu = n_gpu[:, ~exclude][:, None, :]
        n_ref = n_ref[:, ~exclude][:, None, :]
    zg = np.all(n_gpu == 0, axis=0)
    zr = np.all(n_ref == 0, axis=0)
    assert np.array_equal(zg, zr), f"invalid masks differ at {np.argwhere(zg != zr)[:5]}"
    ang = _angle(n_gpu[:, ~zr], n_ref[:, ~zr])
    assert ang.size == 0 or ang.max() <= ANG_TOL, ang.max()
    if ang.size:
        assert np.abs(np.linalg.norm(n_gpu[:, ~zr], axis=0) - 1).max() < 1e-5
    return float(ang.max()) if ang.size else 0.0


def _check_depth(d_gpu, d_in, d_ref):
    valid = (d_in > 0) & np.isfinite(d_in)
    assert d_gpu[~valid].tobytes() == d_in[~valid].tobytes(), "invalid pixels must be copied bitwise"
    err = np.abs(d_gpu[valid].astype(np.float64) - d_ref[valid].astype(np.float64))
    assert err.size == 0 or err.max() <= ADF_TOL, err.max()
    return float(err.max()) if err.size else 0.0


FRAMES = [
    ("C1", {}), ("C1n", {}), ("C1n", {"holes": 0.02}), ("C2", {}), ("C2", {"holes": 0.01}),
    ("C2", {"W": 333, "H": 251}), ("RAMP", {}),
]


@pytest.mark.parametrize("name,kw", FRAMES)
def test_adf_and_fused_normals(pm, name, kw):
    fr = scenegen.make_config(name, **kw)
    iters = fr["iters"] if name != "RAMP" else 7
    d_in = fr["depth"].numpy()
    d_out, nrm = pm.adf_filter(fr["depth"].to(DEV), fr["K"], fr["lam"], fr["kappa"], iters)
    torch.cuda.synchronize()
    d_gpu = d_out.cpu().numpy()
    _check_depth(d_gpu, d_in, oracle.adf(d_in, fr["lam"], fr["kappa"], iters))
    # fused normals against the oracle's normals of the GPU's own filtered depth
    _check_normals(nrm.cpu().numpy(), oracle.normals(d_gpu, fr["K"]))


@pytest.mark.parametrize("name,kw", FRAMES)
def test_normals_standalone(pm, name, kw):
    fr = scenegen.make_config(name, **kw)
    n = pm.normals_from_depth(fr["depth"].to(DEV), fr["K"])
    torch.cuda.synchronize()
    _check_normals(n.cpu().numpy(), oracle.normals(fr["depth"].numpy(), fr["K"]))


def test_adf_special_values_and_edges(pm):
    # NaN / inf / negative / zero pixels copied bitwise; N = 0 copies the
    # input; a constant image is a bitwise fixed point (P4)
    rng = np.random.default_rng(0)
    d = (1.0 + 0.01 * rng.standard_normal((37, 45))).astype(np.float32)
    d[3, 4], d[10, 10], d[20, 0], d[36, 44], d[0, 0] = np.nan, np.inf, -2.0, 0.0, -0.0
    K = scenegen.intrinsics_for(45, 37)
    for it in (0, 1, 5, 13):
        out, nrm = pm.adf_filter(torch.from_numpy(d).to(DEV), K, 0.2, 0.02, it)
        torch.cuda.synchronize()
        _check_depth(out.cpu().numpy(), d, oracle.adf(d, 0.2, 0.02, it))
        _check_normals(nrm.cpu().numpy(), oracle.normals(out.cpu().numpy(), K))
    c = torch.full((33, 70), 1.25, device=DEV)
    out, _ = pm.adf_filter(c, K, 0.25, 0.03, 30)
    assert torch.equal(out, c)


def test_adf_lambda_quarter_spike_and_tiny_depths(pm):
    """lambda = 1/4, a spike over much smaller (valid) neighbours: c = 1,
    lambda c = 1/4 and in f32 the update C + lc*lap rounds to 0 (the
    neighbour sum is below half an ulp of 4C).  Validity is fixed by the
    input (Q4) and carried across passes: for lambda > 0.249 a valid pixel's
    update is floored at 2^-149 (adf_cell.cuh keep_valid), so the spike stays
    valid (the fp64 oracle gives ~1e-8) and later passes keep diffusing it.
    The fused normals must equal the oracle's normals of the GPU's own depth.
    Tiny valid depths (< 2^-100) run the checked sweeps."""
    K = scenegen.intrinsics_for(40, 30)
    d = np.full((30, 40), 1e-8, np.float32)
    d[12, 17] = 1.0
    d[5, 30] = 2.0
    for iters, T in ((1, 4), (2, 4), (3, 1), (6, 4), (9, 2)):
        for eng in (pm.ENGINE_TILED, pm.ENGINE_REG):
            out, nrm = pm.adf_filter(torch.from_numpy(d).to(DEV), K, 0.25, 0.03, iters, iters_per_pass=T, engine=eng)
            torch.cuda.synchronize()
            o = out.cpu().numpy()
            _check_depth(o, d, oracle.adf(d, 0.25, 0.03, iters))
            assert np.all(o > 0) and np.all(np.isfinite(o)), "validity must be carried (every input is valid)"
            if iters == 1:
                assert 0.0 < o[12, 17] <= 1e-7 and 0.0 < o[5, 30] <= 1e-7
            # known f32 limit: a window holding a depth below
            # ~1e-19 m underflows |m|^2 in f32 and reads invalid, while the
            # fp64 oracle still returns a normal -- those windows are excluded
            tiny = o < 1e-19
            ex = np.zeros_like(tiny)
            for dy in (-1, 0, 1):
                for dx in (-1, 0, 1):
                    ex |= np.roll(np.roll(tiny, dy, 0), dx, 1)
            n_np = nrm.cpu().numpy()
            assert np.all(np.isfinite(n_np))
            _check_normals(n_np, oracle.normals(o, K), exclude=ex)
    t = (1.0 + 0.01 * np.random.default_rng(4).standard_normal((30, 40))).astype(np.float32)
    t[3:9, 4:11] = 1e-35
    out, _ = pm.adf_filter(torch.from_numpy(t).to(DEV), K, 0.15, 0.03, 9, normals=False)
    torch.cuda.synchronize()
    _check_depth(out.cpu().numpy(), t, oracle.adf(t, 0.15, 0.03, 9))


def test_adf_validity_carried_across_passes_with_holes(pm):
    """holes plus zeroed-out spikes at lambda = 1/4 over several
    passes: the output is valid exactly where the input is (Q4), for every
    blocking depth, and within tolerance of the oracle."""
    fr = scenegen.make_config("C2", W=128, H=96, holes=0.02)
    d = fr["depth"].numpy().copy()
    d[40:44, 60:64] = 1e-9        # valid, far below the neighbours: the spike pattern inverted
    d[10, 10] = 50.0              # a spike that rounds to its neighbours' scale
    valid_in = (d > 0) & np.isfinite(d)
    ref = oracle.adf(d, 0.25, 0.03, 13)
    for T in (1, 3, 4, 13):
        for eng in (pm.ENGINE_TILED, pm.ENGINE_REG):
            out, _ = pm.adf_filter(torch.from_numpy(d).to(DEV), fr["K"], 0.25, 0.03, 13, iters_per_pass=T,
                                   engine=eng, normals=False)
            torch.cuda.synchronize()
            o = out.cpu().numpy()
            assert np.array_equal((o > 0) & np.isfinite(o), valid_in), (T, eng)
            _check_depth(o, d, ref)


def test_adf_bitwise_invariance_to_blocking_and_batch(pm):
    # identical arithmetic per sweep -> bitwise independent of
    # the iterations fused per pass and of batching
    fr = scenegen.make_config("C2", W=320, H=240)
    d = fr["depth"].to(DEV)
    ref, nref = pm.adf_filter(d, fr["K"], fr["lam"], fr["kappa"], 17, iters_per_pass=1)
    for T in (2, 3, 4, 5, 8, 16):
        out, nrm = pm.adf_filter(d, fr["K"], fr["lam"], fr["kappa"], 17, iters_per_pass=T)
        assert torch.equal(out, ref), T
        assert torch.equal(nrm, nref), T
    batch = torch.stack([d, d.flip(0), d])
    out, nrm = pm.adf_filter(batch.contiguous(), fr["K"], fr["lam"], fr["kappa"], 17)
    assert torch.equal(out[0], ref) and torch.equal(out[2], ref) and torch.equal(nrm[2], nref)
    o1, _ = pm.adf_filter(d.flip(0).contiguous(), fr["K"], fr["lam"], fr["kappa"], 17)
    assert torch.equal(out[1], o1)


def _ransac_compare(pm, depth_np, labels_np, K, R, H, tau, seed, frame_id=0, sampler=0, select=0):
    planes, counts, errq = pm.ransac_planes(torch.from_numpy(depth_np).to(DEV), K,
                                            torch.from_numpy(labels_np).to(DEV), R, H, tau, seed,
                                            first_frame_id=frame_id, sampler=sampler, select=select, debug=True)
    torch.cuda.synchronize()
    ref = oracle.ransac(depth_np, labels_np, K, R, H, tau, seed, frame_id=frame_id, sampler=sampler,
                        select=select, debug=True)
    cg = counts.cpu().numpy()
    assert np.array_equal(cg, ref["counts"]), "per-hypothesis inlier counts must be bit-exact"
    assert np.array_equal(errq.cpu().numpy().view(np.uint64), ref["errq_all"]), "fixed-point error sums"
    assert np.array_equal(planes.n_points.cpu().numpy(), ref["n_points"])
    assert np.array_equal(planes.best_hyp.cpu().numpy(), ref["best_hyp"])
    assert np.array_equal(planes.status.cpu().numpy(), ref["status"])
    assert np.array_equal(planes.inliers.cpu().numpy(), ref["inliers"])
    ok = ref["status"] <= 1
    if ok.any():
        assert np.abs(planes.n.cpu().numpy()[ok] - ref["n"][ok]).max() <= REFIT_TOL
        assert np.abs(planes.d.cpu().numpy()[ok] - ref["d"][ok]).max() <= REFIT_TOL
        assert np.abs(planes.centroid.cpu().numpy()[ok] - ref["centroid"][ok]).max() <= REFIT_TOL
        # the refit's own fixed-point error sum, exact: sum_dist = f32(errq[best] * 2^-24)
        sd = planes.sum_dist.cpu().numpy()[ok]
        want = (ref["errq"][ok].astype(np.float64) / 2**24).astype(np.float32)
        assert np.array_equal(sd, want)
    return ref


@pytest.mark.parametrize("name,kw,filtered", [
    ("C1", {}, False), ("C1n", {}, True), ("C1n", {"holes": 0.02}, True), ("C2", {}, False),
    ("C2", {}, True), ("C2", {"holes": 0.01}, True), ("C2", {"W": 333, "H": 251}, True)])
def test_ransac_bit_exact(pm, name, kw, filtered):
    fr = scenegen.make_config(name, **kw)
    d = fr["depth"]
    if filtered:                                  # the GPU-filtered frame, shared by both sides
        d, _ = pm.adf_filter(d.to(DEV), fr["K"], fr["lam"], fr["kappa"], fr["iters"], normals=False)
        d = d.cpu()
    _ransac_compare(pm, d.numpy(), fr["labels"].numpy(), fr["K"], fr["n_regions"], fr["n_hyp"], fr["tau"],
                    fr["seed"])


@pytest.mark.parametrize("n_hyp", [1, 3, 8, 16, 33, 64, 100, 129, 256, 700, 2100])
def test_ransac_counts_default_kernel_every_layout(pm, n_hyp):
    """Counts of the default scoring kernel (no error sums: packed FFMA2 pairs
    for even K) bit-exact against the oracle for every (K, L) layout the
    launcher picks (n_hyp 1..2100 -> K in {1, 2, 4, 8, 16}, L in 8..256)."""
    fr = scenegen.make_config("C2", W=200, H=150)
    d, lab = fr["depth"].numpy(), fr["labels"].numpy()
    R = 6
    lab = np.where(lab >= 0, lab % R, -1).astype(np.int32)
    planes, counts, errq = pm.ransac_planes(torch.from_numpy(d).to(DEV), fr["K"], torch.from_numpy(lab).to(DEV), R,
                                            n_hyp, fr["tau"], 5, debug="counts")
    torch.cuda.synchronize()
    assert errq is None
    ref = oracle.ransac(d, lab, fr["K"], R, n_hyp, fr["tau"], 5, debug=True)
    assert np.array_equal(counts.cpu().numpy(), ref["counts"])
    assert np.array_equal(planes.best_hyp.cpu().numpy(), ref["best_hyp"])
    assert np.array_equal(planes.inliers.cpu().numpy(), ref["inliers"])
    assert np.array_equal(planes.status.cpu().numpy(), ref["status"])


def test_ransac_noise_free_plane(pm):
    fr = scenegen.make_config("RAMP")
    lab = np.where(fr["depth"].numpy() > 0, 0, -1).astype(np.int32)
    ref = _ransac_compare(pm, fr["depth"].numpy(), lab, fr["K"], 1, 64, fr["tau"], fr["seed"])
    assert ref["status"][0] == 0 and ref["inliers"][0] == ref["n_points"][0]


def test_ransac_enumerate_and_select_error(pm):
    fr = scenegen.make_config("C1n", holes=0.3)
    d = fr["depth"].numpy()
    lab = fr["labels"].numpy().copy()
    # shrink regions to tiny point sets so that ENUMERATE covers all triples
    keep = np.zeros_like(lab, bool)
    keep[::7, ::5] = True
    lab[~keep] = -1
    ref = oracle.ransac(d, lab, fr["K"], 4, 1, fr["tau"], 1)
    nmax = int(ref["n_points"].max())
    _ransac_compare(pm, d, lab, fr["K"], 4, math.comb(nmax, 3), fr["tau"], 1, sampler=1)
    _ransac_compare(pm, d, fr["labels"].numpy(), fr["K"], 4, 64, fr["tau"], 9, select=1)


@pytest.mark.parametrize("name,kw,H", [("C1n", {}, 64), ("C2", {}, 64), ("C2", {"holes": 0.01}, 300),
                                       ("C1n", {}, 1)])
def test_ransac_early_exit_selection(pm, name, kw, H):
    """The *_EARLY select modes (P:292 early exit, Q20) against the oracle's
    sequential loop: best_hyp, status, inliers bit-exact, refit in tolerance
    (the warp's prefix-best scan replays the loop, chunks of 32 hypotheses)."""
    fr = scenegen.make_config(name, **kw)
    d, lab = fr["depth"].numpy(), fr["labels"].numpy()
    for sel in (pm.SELECT_COUNT_EARLY, pm.SELECT_ERROR_EARLY):
        _ransac_compare(pm, d, lab, fr["K"], 4, H, fr["tau"], 11, select=sel)


def test_ransac_frame_ids_and_batch_invariance(pm):
    d, lab, K = scenegen.stair_stream(10, 3, W=160, H=120, n_regions=16)
    planes = pm.ransac_planes(d.to(DEV), K, lab.to(DEV), 16, 32, 0.01, 77, first_frame_id=10)
    torch.cuda.synchronize()
    for i in range(3):
        ref = oracle.ransac(d[i].numpy(), lab[i].numpy(), K, 16, 32, 0.01, 77, frame_id=10 + i)
        assert np.array_equal(planes.best_hyp[i].cpu().numpy(), ref["best_hyp"])
        assert np.array_equal(planes.inliers[i].cpu().numpy(), ref["inliers"])
        single = pm.ransac_planes(d[i].contiguous().to(DEV), K, lab[i].contiguous().to(DEV), 16, 32, 0.01, 77,
                                  first_frame_id=10 + i)
        assert torch.equal(single.raw, planes.raw[i])


def test_ransac_batched_odd_frame_size(pm):
    """W*H odd: frames 1 and 2 of the batch start 8 B off a 16-B boundary in
    the compacted point buffer (the refit's bulk copies round the span down /
    up); every frame must still equal the oracle and its single-frame call."""
    d, lab, K = scenegen.stair_stream(40, 3, W=333, H=251, n_regions=16)
    planes = pm.ransac_planes(d.to(DEV), K, lab.to(DEV), 16, 64, 0.01, 5, first_frame_id=40)
    torch.cuda.synchronize()
    for i in range(3):
        ref = oracle.ransac(d[i].numpy(), lab[i].numpy(), K, 16, 64, 0.01, 5, frame_id=40 + i)
        assert np.array_equal(planes.best_hyp[i].cpu().numpy(), ref["best_hyp"])
        assert np.array_equal(planes.inliers[i].cpu().numpy(), ref["inliers"])
        assert np.array_equal(planes.status[i].cpu().numpy(), ref["status"])
        ok = ref["status"] <= 1
        assert np.abs(planes.n[i].cpu().numpy()[ok] - ref["n"][ok]).max() <= REFIT_TOL
        assert np.abs(planes.centroid[i].cpu().numpy()[ok] - ref["centroid"][ok]).max() <= REFIT_TOL
        single = pm.ransac_planes(d[i].contiguous().to(DEV), K, lab[i].contiguous().to(DEV), 16, 64, 0.01, 5,
                                  first_frame_id=40 + i)
        assert torch.equal(single.raw, planes.raw[i])


def test_ransac_far_outliers_error_sum(pm):
    """Depth scattered over 0.3-6 m in every region: most point-plane distances
    exceed 0.5 m (fixed-point error terms >= 2^23, the refit's second rounding
    branch) and many exceed the 64 m clamp's scale; counts, winner and the
    exact error sum must equal the oracle's."""
    rng = np.random.default_rng(123)
    K = scenegen.intrinsics_for(96, 72)
    depth = rng.uniform(0.3, 6.0, (72, 96)).astype(np.float32)
    labels = (np.arange(96)[None, :] // 24 + 4 * (np.arange(72)[:, None] // 36)).astype(np.int32)
    _ransac_compare(pm, depth, labels, K, 8, 64, 0.02, 3)


def test_ransac_degenerate_cases(pm):
    K = scenegen.intrinsics_for(64, 48)
    depth = np.full((48, 64), 1.5, np.float32)
    lab = np.full((48, 64), -1, np.int32)
    lab[3, 4] = lab[7, 9] = 0                  # 2 points -> TOO_FEW
    lab[10, 5:20] = 1                          # collinear -> DEGENERATE
    lab[20:30, 20:30] = 3                      # plane -> OK
    lab[40, 40] = 99                           # out-of-range label: ignored
    ref = _ransac_compare(pm, depth, lab, K, 5, 16, 0.01, 1)
    assert list(ref["status"]) == [2, 3, 2, 0, 2]


def test_ransac_many_regions_per_chunk(pm):
    """Hundreds of 4x4-pixel regions (some empty, some with 1-2 points) so one
    8192-point score / refit chunk meets far more than 32 regions: the refit's
    per-region prefetch (first 31 regions of a chunk by shuffle, the rest by
    direct loads) and the 32-ary first-region search, bit-exact vs the oracle."""
    fr = scenegen.make_config("C2", W=128, H=96)
    d = fr["depth"].numpy()
    v, u = np.mgrid[0:96, 0:128]
    lab = ((v // 4) * 32 + u // 4).astype(np.int32)          # 768 regions of 16 px
    lab[(lab % 7) == 3] = -1                                  # empty regions
    lab[((lab % 11) == 5) & ((u % 4) > 0)] = -1               # 4-point regions
    lab[((lab % 13) == 6) & ((u % 4) + (v % 4) > 0)] = -1     # 1-point regions
    ref = _ransac_compare(pm, d, lab, fr["K"], 768, 16, fr["tau"], 3)
    assert (ref["n_points"] == 0).any() and (ref["n_points"] == 1).any() and (ref["status"] == 0).any()


def test_pipeline_mixed_hole_frames_equal_separate_calls(pm):
    """pm_process_frames on a batch mixing hole-free frames, frames with
    dropout holes and a frame with a tiny (< 2^-100) depth equals
    adf_filter + ransac_planes exactly, for lambda under and over 0.249 and
    for one and several ADF passes."""
    d, lab, K = scenegen.stair_stream(7, 5, W=160, H=120, n_regions=16)
    d = d.clone()
    rng = np.random.default_rng(11)
    for i in (1, 3):
        m = torch.from_numpy(rng.random((120, 160)) < 0.02)
        d[i][m] = 0.0
    d[4][60, 80] = 1e-35
    dev = torch.device(DEV)
    for lam, iters in ((0.15, 20), (0.25, 9), (0.15, 3)):
        d_out, nrm, planes = pm.process_frames(d.to(dev), lab.to(dev), K, lam, 0.03, iters, 16, 64, 0.01, 21,
                                               first_frame_id=7)
        ref_d, ref_n = pm.adf_filter(d.to(dev), K, lam, 0.03, iters)
        ref_p = pm.ransac_planes(ref_d, K, lab.to(dev), 16, 64, 0.01, 21, first_frame_id=7)
        torch.cuda.synchronize()
        assert torch.equal(d_out, ref_d) and torch.equal(nrm, ref_n)
        assert torch.equal(planes.raw, ref_p.raw), (lam, iters)


@pytest.mark.parametrize("W,H", [(3, 3), (5, 4), (7, 33), (31, 9), (33, 3)])
def test_pipeline_tiny_frames(pm, W, H):
    """Frames at and just above the minimum size (3x3) and narrower than a
    warp: partial tiles everywhere, the compaction's per-step coordinate
    advance wrapping several rows at once (W < 32), one to few points per
    region.  Depth, normals and planes of pm_process_frames vs the oracle,
    batched frames vs single-frame calls."""
    rng = np.random.default_rng(W * 100 + H)
    K = scenegen.intrinsics_for(W, H)
    B, R = 3, 4
    d = (1.0 + 0.3 * rng.random((B, H, W))).astype(np.float32)
    d[1, 0, 0] = 0.0
    lab = rng.integers(-1, R, (B, H, W)).astype(np.int32)
    dev = torch.device(DEV)
    for iters in (0, 3, 9):
        d_out, nrm, planes = pm.process_frames(torch.from_numpy(d).to(dev), torch.from_numpy(lab).to(dev), K, 0.15,
                                               0.03, iters, R, 16, 0.05, 3, first_frame_id=2)
        torch.cuda.synchronize()
        for i in range(B):
            o = d_out[i].cpu().numpy()
            _check_depth(o, d[i], oracle.adf(d[i], 0.15, 0.03, iters))
            _check_normals(nrm[i].cpu().numpy(), oracle.normals(o, K))
            ref = oracle.ransac(o, lab[i], K, R, 16, 0.05, 3, frame_id=2 + i)
            assert np.array_equal(planes.n_points[i].cpu().numpy(), ref["n_points"])
            assert np.array_equal(planes.best_hyp[i].cpu().numpy(), ref["best_hyp"])
            assert np.array_equal(planes.inliers[i].cpu().numpy(), ref["inliers"])
            assert np.array_equal(planes.status[i].cpu().numpy(), ref["status"])


def test_pipeline_no_regions_and_unlabelled(pm):
    """n_regions = 0 (RANSAC skipped: depth and normals still produced) and
    every label -1 (every region TOO_FEW with 0 points)."""
    fr = scenegen.make_config("C1n")
    dev = torch.device(DEV)
    d = fr["depth"].to(dev)
    d_out, nrm, planes = pm.process_frames(d, fr["labels"].to(dev), fr["K"], fr["lam"], fr["kappa"], fr["iters"],
                                           0, fr["n_hyp"], fr["tau"], fr["seed"])
    ref_d, ref_n = pm.adf_filter(d, fr["K"], fr["lam"], fr["kappa"], fr["iters"])
    torch.cuda.synchronize()
    assert torch.equal(d_out, ref_d) and torch.equal(nrm, ref_n)
    none = torch.full_like(fr["labels"], -1).to(dev)
    _, _, planes = pm.process_frames(d, none, fr["K"], fr["lam"], fr["kappa"], fr["iters"], 4, fr["n_hyp"],
                                     fr["tau"], fr["seed"])
    torch.cuda.synchronize()
    assert planes.n_points.cpu().tolist() == [0, 0, 0, 0]
    assert planes.status.cpu().tolist() == [2, 2, 2, 2]


def test_pipeline_end_to_end(pm):
    fr = scenegen.make_config("C2")
    dev = torch.device(DEV)
    d_out, nrm, planes = pm.process_frames(fr["depth"].to(dev), fr["labels"].to(dev), fr["K"], fr["lam"],
                                           fr["kappa"], fr["iters"], fr["n_regions"], fr["n_hyp"], fr["tau"],
                                           fr["seed"])
    torch.cuda.synchronize()
    d_gpu = d_out.cpu().numpy()
    ref = oracle.ransac(d_gpu, fr["labels"].numpy(), fr["K"], fr["n_regions"], fr["n_hyp"], fr["tau"], fr["seed"])
    assert np.array_equal(planes.best_hyp.cpu().numpy(), ref["best_hyp"])
    assert np.array_equal(planes.status.cpu().numpy(), ref["status"])
    assert (ref["status"] == 0).mean() > 0.9


# --------------------------------------------------------------------------
# BASELINE.json full-size configurations, in the launch configuration the
# bench uses, checked on samples the oracle can compute.
def _crop_adf_check(pm, d_in, d_gpu, lam, kappa, iters, rng, n=6, size=48):
    """ADF is local: after N sweeps a pixel depends only on pixels within N
    (L1) of it, so the oracle on a crop with an N-pixel margin reproduces the
    crop's centre exactly (the crop border acts as a zero-flux edge only for
    pixels that are discarded)."""
    H, W = d_in.shape
    m = iters
    for _ in range(n):
        y = int(rng.integers(0, max(1, H - size)))
        x = int(rng.integers(0, max(1, W - size)))
        y0, x0 = max(0, y - m), max(0, x - m)
        y1, x1 = min(H, y + size + m), min(W, x + size + m)
        ref = oracle.adf(np.ascontiguousarray(d_in[y0:y1, x0:x1]), lam, kappa, iters)
        cy0, cx0 = y - y0, x - x0
        sub_ref = ref[cy0:cy0 + size, cx0:cx0 + size]
        sub_in = d_in[y:y + size, x:x + size]
        _check_depth(d_gpu[y:y + size, x:x + size], sub_in, sub_ref)


@pytest.mark.parametrize("name", ["C3", "C5"])
def test_full_size_configs_sampled(pm, name):
    fr = scenegen.make_config(name)
    rng = np.random.default_rng(42)
    d_in = fr["depth"].numpy()
    dev_d = fr["depth"].to(DEV)
    d_out, nrm = pm.adf_filter(dev_d, fr["K"], fr["lam"], fr["kappa"], fr["iters"])
    torch.cuda.synchronize()
    d_gpu = d_out.cpu().numpy()
    _crop_adf_check(pm, d_in, d_gpu, fr["lam"], fr["kappa"], fr["iters"], rng)
    # normals: oracle on crops of the GPU depth (+1 margin), compared on the centre
    n_gpu = nrm.cpu().numpy()
    H, W = d_gpu.shape
    for _ in range(6):
        y, x = int(rng.integers(0, H - 64)), int(rng.integers(0, W - 64))
        y0, x0, y1, x1 = max(0, y - 1), max(0, x - 1), min(H, y + 65), min(W, x + 65)
        ref = oracle.normals(np.ascontiguousarray(d_gpu[y0:y1, x0:x1]), scenegen.Intrinsics(
            fr["K"].fx, fr["K"].fy, fr["K"].cx - x0, fr["K"].cy - y0))
        cy, cx = y - y0, x - x0
        _check_normals(n_gpu[:, y:y + 64, x:x + 64], ref[:, cy:cy + 64, cx:cx + 64])
    # RANSAC over every region of the full frame (GPU-filtered depth), bit-exact
    _ransac_compare(pm, d_gpu, fr["labels"].numpy(), fr["K"], fr["n_regions"], fr["n_hyp"], fr["tau"], fr["seed"])


def test_bench_configuration_sampled(pm):
    """The bench's workload (C4 stream, 512 frames per call, pm_process_frames):
    frames 0, 511 and one in between checked against the oracle."""
    import bench
    B = 512
    first, _ = bench.shard(0, B)
    d, lab, K = scenegen.stair_stream(first, B, bench.W, bench.H, bench.REGIONS, device=DEV)
    d_out, nrm, planes = pm.process_frames(d, lab, K, bench.LAM, bench.KAPPA, bench.ITERS, bench.REGIONS,
                                           bench.HYPS, bench.TAU, bench.SEED, first_frame_id=first)
    torch.cuda.synchronize()
    rng = np.random.default_rng(7)
    for i in [0, int(rng.integers(1, B - 1)), B - 1]:
        d_in = d[i].cpu().numpy()
        d_gpu = d_out[i].cpu().numpy()
        _check_depth(d_gpu, d_in, oracle.adf(d_in, bench.LAM, bench.KAPPA, bench.ITERS))
        _check_normals(nrm[i].cpu().numpy(), oracle.normals(d_gpu, K))
        ref = oracle.ransac(d_gpu, lab[i].cpu().numpy(), K, bench.REGIONS, bench.HYPS, bench.TAU, bench.SEED,
                            frame_id=first + i)
        assert np.array_equal(planes.best_hyp[i].cpu().numpy(), ref["best_hyp"])
        assert np.array_equal(planes.inliers[i].cpu().numpy(), ref["inliers"])
        assert np.array_equal(planes.status[i].cpu().numpy(), ref["status"])
        ok = ref["status"] <= 1
        assert np.abs(planes.n[i].cpu().numpy()[ok] - ref["n"][ok]).max() <= REFIT_TOL
        assert np.abs(planes.centroid[i].cpu().numpy()[ok] - ref["centroid"][ok]).max() <= REFIT_TOL


# -------------------------------------------------- NEXT-1 paper-literal modes
@pytest.mark.parametrize("name,kw", [("C1n", {}), ("C2", {}), ("C2", {"holes": 0.01}), ("C2", {"W": 333, "H": 251})])
def test_divergence_scheme_and_printed_normals(pm, name, kw):
    fr = scenegen.make_config(name, **kw)
    d_in = fr["depth"].numpy()
    d_out, nrm = pm.adf_filter(fr["depth"].to(DEV), fr["K"], fr["lam"], fr["kappa"], fr["iters"],
                               scheme=pm.ADF_DIVERGENCE, normals_mode=pm.NORMALS_AS_PRINTED)
    torch.cuda.synchronize()
    d_gpu = d_out.cpu().numpy()
    _check_depth(d_gpu, d_in, oracle.adf(d_in, fr["lam"], fr["kappa"], fr["iters"], scheme=oracle.ADF_DIVERGENCE))
    _check_normals(nrm.cpu().numpy(), oracle.normals(d_gpu, fr["K"], mode=oracle.NORMALS_AS_PRINTED))
    n2 = pm.normals_from_depth(fr["depth"].to(DEV), fr["K"], mode=pm.NORMALS_AS_PRINTED)
    torch.cuda.synchronize()
    _check_normals(n2.cpu().numpy(), oracle.normals(d_in, fr["K"], mode=oracle.NORMALS_AS_PRINTED))
    # blocking invariance holds for this scheme too
    d2, _ = pm.adf_filter(fr["depth"].to(DEV), fr["K"], fr["lam"], fr["kappa"], fr["iters"], iters_per_pass=3,
                          scheme=pm.ADF_DIVERGENCE, normals=False)
    assert torch.equal(d2.cpu(), d_out.cpu())


def test_host_pipeline_matches_device_pipeline(pm):
    """pm_process_frames_host (chunked, double-buffered, sensor-native uint16
    inputs) gives bit-identical plane tables to pm_process_frames on the same
    frames converted on the device."""
    B, W, H, R, NH = 5, 160, 120, 16, 32
    d, lab, K = scenegen.stair_stream(100, B, W, H, R)
    mm = torch.round(d.double() * 1000).clamp(0, 65535).to(torch.int32).to(torch.uint16)
    lab16 = torch.where(lab < 0, torch.full_like(lab, 0xFFFF), lab).to(torch.int32).to(torch.uint16)
    depth_out = torch.empty(B, H, W).pin_memory()
    normals_out = torch.empty(B, 3, H, W).pin_memory()
    planes_h = pm.process_frames_host(mm.pin_memory(), lab16.pin_memory(), K, 0.15, 0.03, 20, R, NH, 0.01, 77,
                                      first_frame_id=100, chunk_frames=2, depth_out=depth_out,
                                      normals_out=normals_out)
    dm = pm.depth_u16_to_metres(mm.to(DEV))
    d_dev, n_dev, planes_d = pm.process_frames(dm, lab.to(DEV), K, 0.15, 0.03, 20, R, NH, 0.01, 77,
                                               first_frame_id=100)
    torch.cuda.synchronize()
    assert torch.equal(planes_h.raw, planes_d.raw.cpu())
    assert torch.equal(depth_out, d_dev.cpu()) and torch.equal(normals_out, n_dev.cpu())
    # f32 / int32 host formats, one chunk
    planes_f = pm.process_frames_host(dm.cpu().contiguous(), lab.contiguous(), K, 0.15, 0.03, 20, R, NH, 0.01, 77,
                                      first_frame_id=100, chunk_frames=8)
    assert torch.equal(planes_f.raw, planes_d.raw.cpu())
    # uint8 labels (0xFF = none), three chunks of 2 + 2 + 1 frames
    lab8 = torch.where(lab < 0, torch.full_like(lab, 0xFF), lab).to(torch.uint8)
    planes_8 = pm.process_frames_host(mm.pin_memory(), lab8.pin_memory(), K, 0.15, 0.03, 20, R, NH, 0.01, 77,
                                      first_frame_id=100, chunk_frames=2)
    assert torch.equal(planes_8.raw, planes_d.raw.cpu())
    # and against the oracle for one frame
    ref = oracle.ransac(d_dev[3].cpu().numpy(), lab[3].numpy(), K, R, NH, 0.01, 77, frame_id=103)
    assert np.array_equal(planes_h.best_hyp[3].numpy(), ref["best_hyp"])
    assert np.array_equal(planes_h.inliers[3].numpy(), ref["inliers"])


# --------------------------------------------- NEXT-2: labels from normals
@pytest.mark.parametrize("name,kw", [("C1n", {}), ("C2", {}), ("C2", {"noise": False}), ("C2", {"holes": 0.01}),
                                     ("C2", {"W": 333, "H": 251}), ("C3", {})])
def test_segment_regions_bit_exact(pm, name, kw):
    fr = scenegen.make_config(name, **kw)
    d_out, nrm = pm.adf_filter(fr["depth"].to(DEV), fr["K"], fr["lam"], fr["kappa"], fr["iters"])
    min_area = 300 if fr["W"] >= 320 else 20
    labels, nreg, edges = pm.segment_regions(nrm, 30, 90, min_area, 1024, edges=True)
    torch.cuda.synchronize()
    ref_lab, ref_n, ref_e = oracle.segment_regions(nrm.cpu().numpy(), 30, 90, min_area, 1024)
    assert np.array_equal(edges.cpu().numpy(), ref_e)
    assert int(nreg[0]) == ref_n
    assert np.array_equal(labels.cpu().numpy(), ref_lab)


def test_segment_then_ransac_pipeline(pm):
    """depth -> ADF + normals -> segmentation -> RANSAC, all on the device,
    batched; bit-exact against the oracle chain on the GPU's buffers."""
    d, _, K = scenegen.stair_stream(40, 3, 320, 240, 8)
    dev_d = d.to(DEV)
    d_out, nrm = pm.adf_filter(dev_d, K, 0.15, 0.03, 20)
    labels, nreg, _ = pm.segment_regions(nrm, 30, 90, 200, 64)
    planes = pm.ransac_planes(d_out, K, labels, 64, 64, 0.01, 3, first_frame_id=40)
    torch.cuda.synchronize()
    for i in range(3):
        ref_lab, ref_n, _ = oracle.segment_regions(nrm[i].cpu().numpy(), 30, 90, 200, 64)
        assert np.array_equal(labels[i].cpu().numpy(), ref_lab) and int(nreg[i]) == ref_n
        ref = oracle.ransac(d_out[i].cpu().numpy(), ref_lab, K, 64, 64, 0.01, 3, frame_id=40 + i)
        assert np.array_equal(planes.best_hyp[i].cpu().numpy(), ref["best_hyp"])
        assert np.array_equal(planes.status[i].cpu().numpy(), ref["status"])
        assert (ref["status"][:ref_n] == 0).mean() > 0.5


# ------------------------------------------------------------ NEXT-3 polygons
def _poly_label_images():
    cv2 = pytest.importorskip("cv2")
    ims = []
    fr = scenegen.make_config("C2", noise=False)
    n = oracle.normals(fr["depth"].numpy(), fr["K"]).astype(np.float32)
    lab, nr, _ = oracle.segment_regions(n, 30, 90, 300)
    ims.append((lab, nr, fr))
    rng = np.random.default_rng(4)
    H, W = fr["depth"].shape
    blob = np.full((H, W), -1, np.int32)
    for r in range(12):                               # random ellipses, later ones painted over earlier
        m = np.zeros((H, W), np.uint8)
        cv2.ellipse(m, (int(rng.integers(20, W - 20)), int(rng.integers(20, H - 20))),
                    (int(rng.integers(3, 60)), int(rng.integers(3, 40))), float(rng.uniform(0, 180)), 0, 360, 1, -1)
        blob[m > 0] = r
    ims.append((blob, 12, fr))
    return ims


def test_region_polygons_rasterize_lift_bit_exact(pm):
    for lab, R, fr in _poly_label_images():
        H, W = lab.shape
        labs = np.stack([lab, np.flipud(lab).copy()])          # a batch of two frames
        polys = pm.region_polygons(torch.from_numpy(labs).to(DEV), R, eps=3.0, max_contour=8192, max_vertices=512)
        ras = pm.rasterize_polygons(polys, W, H)
        depth = torch.stack([fr["depth"], fr["depth"].flip(0)]).contiguous().to(DEV)
        planes = pm.ransac_planes(depth, fr["K"], torch.from_numpy(np.where(labs >= 0, labs, -1)).to(DEV), R, 64,
                                  0.01, 3)
        X = pm.lift_polygon_vertices(polys, planes, fr["K"])
        torch.cuda.synchronize()
        K32 = scenegen.Intrinsics(*[float(np.float32(v)) for v in (fr["K"].fx, fr["K"].fy, fr["K"].cx, fr["K"].cy)])
        for b in range(2):
            ref_polys = []
            for r in range(R):
                c = oracle.trace_contour(labs[b], r)
                assert polys.contour_len[b, r].item() == len(c)
                s = oracle.simplify_dp(c, 3.0) if len(c) else np.zeros((0, 2), np.int32)
                m = polys.n_vertices[b, r].item()
                assert m == len(s)
                assert np.array_equal(polys.vertices[b, r, :m].cpu().numpy(), s)
                ref_polys.append(s)
                raw = planes.raw[b, r].cpu().numpy()
                if raw[10] == 0 and m:
                    pl = raw[:4].view(np.float32).astype(np.float64)
                    Xr = oracle.lift_vertices(s, pl, K32)
                    Xg = X[b, r, :m].cpu().numpy()
                    assert np.array_equal(np.isnan(Xg), np.isnan(Xr))
                    ok = ~np.isnan(Xr)
                    assert np.abs(Xg[ok] - Xr[ok]).max(initial=0) <= 1e-12
                else:
                    assert torch.isnan(X[b, r]).all()
            want = oracle.rasterize_polygons([p if len(p) >= 3 else np.zeros((0, 2), np.int32) for p in ref_polys],
                                             W, H)
            assert np.array_equal(ras[b].cpu().numpy(), want)


def test_region_polygons_edge_cases(pm):
    # empty regions, a single pixel, a two-pixel region, a region touching the
    # image border, contour capacity below the traced length
    lab = np.full((40, 50), -1, np.int32)
    lab[5, 5] = 1
    lab[9, 9:11] = 2
    lab[20:40, 0:50] = 4                      # touches three image borders
    polys = pm.region_polygons(torch.from_numpy(lab).to(DEV), 6, eps=1.0, max_contour=4096, max_vertices=64)
    small = pm.region_polygons(torch.from_numpy(lab).to(DEV), 6, eps=1.0, max_contour=16, max_vertices=64)
    ras = pm.rasterize_polygons(polys, 50, 40)
    torch.cuda.synchronize()
    for r in range(6):
        c = oracle.trace_contour(lab, r)
        assert polys.contour_len[r].item() == len(c) == small.contour_len[r].item()
        s = oracle.simplify_dp(c, 1.0) if len(c) else np.zeros((0, 2), np.int32)
        m = polys.n_vertices[r].item()
        assert m == len(s) and np.array_equal(polys.vertices[r, :m].cpu().numpy(), s)
    assert polys.n_vertices[0].item() == 0 and polys.n_vertices[3].item() == 0
    want = oracle.rasterize_polygons([polys.vertices[r, :polys.n_vertices[r].item()].cpu().numpy()
                                      if polys.n_vertices[r].item() >= 3 else np.zeros((0, 2), np.int32)
                                      for r in range(6)], 50, 40)
    assert np.array_equal(ras.cpu().numpy(), want)


# ------------------------------------------------ register-tile engine (adf_reg.cu)
REG_FRAMES = [("C2", {}), ("C2", {"holes": 0.01}), ("C2", {"W": 332, "H": 251}), ("C2", {"W": 132, "H": 128}),
              ("C2", {"W": 644, "H": 131, "holes": 0.003}), ("C3", {}), ("RAMP", {"W": 400, "H": 300})]


@pytest.mark.parametrize("name,kw", REG_FRAMES)
def test_reg_engine_bitwise_equals_tiled(pm, name, kw):
    """The register engine evaluates the identical per-cell expression, so it
    must equal the shared-memory engine bit for bit: every T, both schemes,
    both normal modes, lambda at the stability limit (validity carried).  So
    must the HOLES engine (unchecked walk + fix-up of the cells next to a
    hole, hole lists carried from the first pass)."""
    fr = scenegen.make_config(name, **kw)
    d = fr["depth"].to(DEV)
    it = 9
    for scheme, nmode, lam in [(pm.ADF_ALG1, pm.NORMALS_GEOMETRIC, fr["lam"]),
                               (pm.ADF_DIVERGENCE, pm.NORMALS_GEOMETRIC, fr["lam"]),
                               (pm.ADF_ALG1, pm.NORMALS_AS_PRINTED, fr["lam"]),
                               (pm.ADF_ALG1, pm.NORMALS_GEOMETRIC, 0.25)]:
        ref, nref = pm.adf_filter(d, fr["K"], lam, fr["kappa"], it, scheme=scheme, normals_mode=nmode,
                                  engine=pm.ENGINE_TILED)
        for T in (1, 2, 3, 4, 5, 7, 9):
            for eng in (pm.ENGINE_REG, pm.ENGINE_HOLES):
                out, nrm = pm.adf_filter(d, fr["K"], lam, fr["kappa"], it, scheme=scheme, normals_mode=nmode,
                                         engine=eng, iters_per_pass=T)
                assert torch.equal(out, ref), (scheme, nmode, lam, T, eng)
                assert torch.equal(nrm, nref), (scheme, nmode, lam, T, eng)
    # standalone normals (0 sweeps) and N = 0
    n_reg = pm.normals_from_depth(d, fr["K"])
    out0, n0 = pm.adf_filter(d, fr["K"], fr["lam"], fr["kappa"], 0, engine=pm.ENGINE_REG)
    out0t, n0t = pm.adf_filter(d, fr["K"], fr["lam"], fr["kappa"], 0, engine=pm.ENGINE_TILED)
    assert torch.equal(out0, d) and torch.equal(n0, n0t) and torch.equal(n_reg, n0t)
    torch.cuda.synchronize()
    d_in = fr["depth"].numpy()
    out, nrm = pm.adf_filter(d, fr["K"], fr["lam"], fr["kappa"], fr["iters"])
    _check_depth(out.cpu().numpy(), d_in, oracle.adf(d_in, fr["lam"], fr["kappa"], fr["iters"]))
    _check_normals(nrm.cpu().numpy(), oracle.normals(out.cpu().numpy(), fr["K"]))


def test_reg_engine_batched_stream_equals_tiled(pm):
    """C4 stream frames batched (the bench launch configuration, persistent
    CTAs over many tiles and frames) against the tiled engine."""
    d, _, K = scenegen.stair_stream(5, 24, 640, 480, 64, device=DEV)
    ref, nref = pm.adf_filter(d, K, 0.15, 0.03, 20, engine=pm.ENGINE_TILED)
    out, nrm = pm.adf_filter(d, K, 0.15, 0.03, 20)
    assert torch.equal(out, ref) and torch.equal(nrm, nref)


@pytest.mark.parametrize("frac", [0.0005, 0.01, 0.02, 0.05])
def test_holes_engine_dropout_stream_equals_tiled(pm, frac):
    """PM_ADF_ENGINE_HOLES on C4-size frames with dropout (the fix-up path,
    its per-tile hole lists reused by the later passes, and above ~1.5 % the
    checked-walk fallback) against the tiled engine, bit for bit; the frame
    flags it leaves let the pipeline's compaction skip nothing it must read."""
    d, lab, K = scenegen.stair_stream(40, 6, 640, 480, 64, device=DEV)
    for i in range(d.shape[0]):
        d[i] = scenegen.dropout(d[i], frac, 77 + i, i)
    d[1] = scenegen.stair_stream(46, 1, 640, 480, 64, device=DEV)[0][0]     # one hole-free frame in the batch
    for T in (4, 3, 16):
        ref, nref = pm.adf_filter(d, K, 0.15, 0.03, 20, engine=pm.ENGINE_TILED, iters_per_pass=T)
        out, nrm = pm.adf_filter(d, K, 0.15, 0.03, 20, engine=pm.ENGINE_HOLES, iters_per_pass=T)
        assert torch.equal(out, ref) and torch.equal(nrm.nan_to_num(7.0), nref.nan_to_num(7.0)), (frac, T)


def test_binding_rejects_mismatched_buffers(pm):
    """the binding checks every output / workspace tensor (device,
    dtype, contiguity, element count) and the labels' shape before calling
    the C ABI, which trusts its pointers."""
    d, lab, K = scenegen.stair_stream(0, 2, 128, 96, 8, device=DEV)
    bad = [dict(depth_out=torch.empty(2, 96, 127, device=DEV)),
           dict(normals_out=torch.empty(2, 3, 96, 128, device=DEV, dtype=torch.float64)),
           dict(planes_out=torch.empty(2, 8, 12, dtype=torch.int32)),                       # host memory
           dict(planes_out=torch.empty(2, 12, 8, dtype=torch.int32, device=DEV).transpose(1, 2)),   # not contiguous
           dict(workspace=torch.empty(10, dtype=torch.float32, device=DEV))]
    for kw in bad:
        with pytest.raises(pm.PMError):
            pm.process_frames(d, lab, K, 0.15, 0.03, 4, 8, 16, 0.01, 1, **kw)
    with pytest.raises(pm.PMError):              # [H, W] labels with [B, H, W] depth
        pm.process_frames(d, lab[0].contiguous(), K, 0.15, 0.03, 4, 8, 16, 0.01, 1)
    with pytest.raises(pm.PMError):
        pm.ransac_planes(d, K, lab[:1].contiguous(), 8, 16, 0.01, 1)
    with pytest.raises(pm.PMError):
        pm.adf_filter(d, K, 0.15, 0.03, 4, out=torch.empty(3, 96, 128, device=DEV))
    with pytest.raises(pm.PMError):
        pm.normals_from_depth(d, K, out=torch.empty(2, 3, 96, 128, device=DEV, dtype=torch.float16))
    # well-formed caller buffers are accepted and used
    do = torch.empty_like(d)
    _, _, pl = pm.process_frames(d, lab, K, 0.15, 0.03, 4, 8, 16, 0.01, 1, depth_out=do)
    torch.cuda.synchronize()
    assert pl.raw.shape == (2, 8, 12) and torch.isfinite(do).all()


def test_host_pipeline_rejects_bad_arguments_before_copying(pm):
    """pm_process_frames_host checks every argument before it
    queues the first copy (and drains its streams on any exit), so a failed
    call leaves nothing in flight and the next call works."""
    d, lab, K = scenegen.stair_stream(0, 3, 128, 96, 8)
    mm = torch.round(d.double() * 1000).to(torch.int32).to(torch.uint16).pin_memory()
    lab8 = torch.where(lab < 0, torch.full_like(lab, 0xFF), lab).to(torch.uint8).pin_memory()
    for bad in (dict(lam=0.3), dict(kappa=-1.0), dict(iters=-1), dict(n_hyp=0), dict(tau=0.0)):
        kw = dict(lam=0.15, kappa=0.03, iters=20, n_hyp=16, tau=0.01)
        kw.update(bad)
        with pytest.raises(pm.PMError):
            pm.process_frames_host(mm, lab8, K, kw["lam"], kw["kappa"], kw["iters"], 8, kw["n_hyp"], kw["tau"], 1,
                                   chunk_frames=1)
    good = pm.process_frames_host(mm, lab8, K, 0.15, 0.03, 20, 8, 16, 0.01, 1, chunk_frames=1)
    dd = pm.depth_u16_to_metres(mm.cuda())
    ref = pm.process_frames(dd, lab.cuda(), K, 0.15, 0.03, 20, 8, 16, 0.01, 1)[2]
    torch.cuda.synchronize()
    assert torch.equal(good.raw, ref.raw.cpu())


def test_host_pipeline_run_length_labels(pm):
    """PM_LABELS_RUNS: the same label image as row runs gives the same plane
    tables (bitwise) as the dense uint8 labels, over chunk boundaries; a row
    whose runs fall short of W leaves the rest unlabelled, runs past W are cut."""
    d, lab, K = scenegen.stair_stream(7, 5, 256, 120, 24)
    mm = torch.round(d.double() * 1000).to(torch.int32).to(torch.uint16).pin_memory()
    lab = lab.clone()
    lab[1, 10:20, 30:90] = -1                                   # unlabelled holes inside a region
    lab[3, :, 200:] = 23                                        # a column band: many short runs
    lab8 = torch.where(lab < 0, torch.full_like(lab, 0xFF), lab).to(torch.uint8).pin_memory()
    runs = pm.encode_label_runs(lab).pin_memory()
    assert runs.nbytes < lab8.numel() // 10
    for chunk in (1, 2, 5):
        dense = pm.process_frames_host(mm, lab8, K, 0.15, 0.03, 20, 24, 32, 0.01, 5, first_frame_id=7,
                                       chunk_frames=chunk)
        rl = pm.process_frames_host(mm, runs, K, 0.15, 0.03, 20, 24, 32, 0.01, 5, first_frame_id=7,
                                    chunk_frames=chunk)
        assert torch.equal(dense.raw, rl.raw), chunk
    # malformed rows: row 0 of frame 0 sums to W - 16 (tail unlabelled); row 1 to W + 40 (cut)
    rs = runs.row_start.clone().numpy().view(np.uint32).astype(np.int64)
    rr = runs.runs.clone().numpy().view(np.uint32).astype(np.int64)
    lab_bad = lab.clone()
    i0 = rs[0]
    rr[i0] = (rr[i0] & 0xFFFF) | (((rr[i0] >> 16) - 16) << 16)
    if rs[1] - rs[0] == 1:
        lab_bad[0, 0, 256 - 16:] = -1
    i1 = rs[2] - 1
    rr[i1] = (rr[i1] & 0xFFFF) | (((rr[i1] >> 16) + 40) << 16)
    bad = pm.LabelRuns(torch.from_numpy(rs.astype(np.uint32).view(np.int32)),
                       torch.from_numpy(rr.astype(np.uint32).view(np.int32)), runs.shape)
    if rs[1] - rs[0] == 1:
        lab_bad8 = torch.where(lab_bad < 0, torch.full_like(lab_bad, 0xFF), lab_bad).to(torch.uint8)
        a = pm.process_frames_host(mm, lab_bad8.pin_memory(), K, 0.15, 0.03, 20, 24, 32, 0.01, 5, chunk_frames=2)
        b = pm.process_frames_host(mm, bad.pin_memory(), K, 0.15, 0.03, 20, 24, 32, 0.01, 5, chunk_frames=2)
        assert torch.equal(a.raw, b.raw)


def test_host_pipeline_async_calls_equal_sync(pm):
    """pm_process_frames_host_async: several calls queued back to back on one
    arena (the next call's uploads run under the previous call's kernels)
    give the tables of the synchronous call, per call."""
    d, lab, K = scenegen.stair_stream(20, 6, 192, 128, 16)
    mm = torch.round(d.double() * 1000).to(torch.int32).to(torch.uint16).pin_memory()
    runs = pm.encode_label_runs(lab).pin_memory()
    dev = torch.device("cuda", 0)
    arena = torch.empty(pm.host_pipeline_arena_bytes(192, 128, 16, 32, 2, pm.DEPTH_U16_MM, pm.LABELS_RUNS),
                        dtype=torch.uint8, device=dev)
    ref = pm.process_frames_host(mm, runs, K, 0.15, 0.03, 20, 16, 32, 0.01, 9, first_frame_id=20, chunk_frames=2,
                                 arena=arena, device=dev)
    outs = [torch.empty(6, 16, pm.PLANE_WORDS, dtype=torch.int32).pin_memory() for _ in range(4)]
    for o in outs:                                   # chunks 2 + 2 + 2: slots 0, 1, 0 -> next call starts on 0
        pm.process_frames_host(mm, runs, K, 0.15, 0.03, 20, 16, 32, 0.01, 9, first_frame_id=20, chunk_frames=2,
                               planes_out=o, arena=arena, device=dev, sync=False)
    torch.cuda.current_stream(dev).synchronize()
    for o in outs:
        assert torch.equal(o, ref.raw)
    with pytest.raises(pm.PMError):
        pm.process_frames_host(mm, runs, K, 0.15, 0.03, 20, 16, 32, 0.01, 9, sync=False)


def test_two_devices_in_one_process(pm):
    """Per-device setup (the kernels' shared-memory attributes are set once per
    device context): process_frames on a second GPU of the same process equals
    the first GPU's result bit for bit.  Needs two visible devices."""
    if torch.cuda.device_count() < 2:
        pytest.skip("needs two CUDA devices")
    d, lab, K = scenegen.stair_stream(0, 2, 128, 96, 16)
    res = []
    for i in (0, 1):
        dev = torch.device("cuda", i)
        out = pm.process_frames(d.to(dev), lab.to(dev), K, 0.15, 0.03, 20, 16, 64, 0.01, 7)
        torch.cuda.synchronize(dev)
        res.append([t.raw.cpu() if hasattr(t, "raw") else t.cpu() for t in out])
    for a, b in zip(*res):
        assert torch.equal(a, b)


def test_auto_engine_after_dropout_and_unaligned_buffers(pm):
    """AUTO after calls that met dropout (it then runs the hole engine) equals
    TILED bit for bit; an output tensor 4 bytes off a 16-byte boundary is
    rejected (the kernels write float4 / bulk-copy rows), labels 4 bytes off
    take the scalar count walk with identical results."""
    d, lab, K = scenegen.stair_stream(60, 4, 640, 480, 64, device=DEV)
    for i in range(4):
        d[i] = scenegen.dropout(d[i], 0.01, 5 + i, i)
    ref, nref = pm.adf_filter(d, K, 0.15, 0.03, 20, engine=pm.ENGINE_TILED)
    for _ in range(3):
        out, nrm = pm.adf_filter(d, K, 0.15, 0.03, 20)
        torch.cuda.synchronize()
        assert torch.equal(out, ref) and torch.equal(nrm.nan_to_num(7.0), nref.nan_to_num(7.0))
    big = torch.empty(d.numel() + 1, device=DEV)
    out_u = big[1:].view(d.shape)                     # 4 bytes past a 16-byte boundary: rejected
    with pytest.raises(pm.PMError):
        pm.adf_filter(d, K, 0.15, 0.03, 20, out=out_u)
    with pytest.raises(pm.PMError):
        pm.normals_from_depth(d, K, out=torch.empty(d.numel() * 3 + 1, device=DEV)[1:].view(4, 3, 480, 640))
    planes = pm.ransac_planes(ref, K, lab, 64, 64, 0.01, 3)
    bl = torch.empty(lab.numel() + 1, dtype=torch.int32, device=DEV)
    lab_u = bl[1:].view(lab.shape)
    lab_u.copy_(lab)
    planes_u = pm.ransac_planes(ref, K, lab_u, 64, 64, 0.01, 3)
    torch.cuda.synchronize()
    assert torch.equal(planes.raw, planes_u.raw)


def test_depth_u16_to_metres_any_alignment(pm):
    """pm_depth_u16_to_metres on views at odd element offsets (input and
    output) equals the aligned conversion: the vector path only runs where
    both addresses allow it."""
    mm = (torch.arange(1003, dtype=torch.int32) * 37 % 65536).to(torch.uint16).to(DEV)
    ref = pm.depth_u16_to_metres(mm)
    for a, b in ((1, 0), (0, 1), (3, 2)):
        src = torch.empty(mm.numel() + a, dtype=torch.uint16, device=DEV)[a:]
        src.copy_(mm)
        dst = torch.empty(mm.numel() + b, device=DEV)[b:]
        out = pm.depth_u16_to_metres(src, out=dst)
        torch.cuda.synchronize()
        assert torch.equal(out, ref)



@pytest.mark.parametrize("H", [16, 64, 200])
def test_ransac_small_region_kernel(pm, H):
    """Frames whose regions average fewer than 512 points score with the
    warp-per-segment kernel (count-only runs: no per-hypothesis error
    requested): per-hypothesis counts, winners, status and inliers bit-exact
    vs the oracle, refit within tolerance."""
    fr = scenegen.make_config("C2", W=320, H=240)
    d = fr["depth"].numpy()
    v, u = np.mgrid[0:240, 0:320]
    lab = ((v // 8) * 40 + u // 8).astype(np.int32)          # 1200 regions of 64 px
    lab[(lab % 17) == 4] = -1
    R = 1200
    planes, counts, _ = pm.ransac_planes(torch.from_numpy(d).to(DEV), fr["K"], torch.from_numpy(lab).to(DEV), R, H,
                                         fr["tau"], 21, debug="counts")
    torch.cuda.synchronize()
    ref = oracle.ransac(d, lab, fr["K"], R, H, fr["tau"], 21, debug=True)
    assert np.array_equal(counts.cpu().numpy(), ref["counts"])
    assert np.array_equal(planes.best_hyp.cpu().numpy(), ref["best_hyp"])
    assert np.array_equal(planes.status.cpu().numpy(), ref["status"])
    assert np.array_equal(planes.inliers.cpu().numpy(), ref["inliers"])
    ok = ref["status"] <= 1
    assert np.abs(planes.n.cpu().numpy()[ok] - ref["n"][ok]).max() <= REFIT_TOL
