"""NEXT-4: the map merge gate (Eqs. 4-5) and the vertical-drift
Kalman filter (Eqs. 6-10), host code in the library (csrc/mapman.cpp) against
the oracle (oracle/mapman.py) and against values fixed by the paper / SPEC
and closed forms.  No GPU: this part of the method runs on the host."""
import math
import random

import numpy as np
import pytest
import torch

from oracle import mapman as orc

pm = pytest.importorskip("paper_2411_01919_b200")


def _row(n, c, inliers=100, status=0):
    """One pm_plane as 12 int32 words (include/pmap.h layout)."""
    f = np.zeros(12, np.float32)
    f[0:3] = n
    f[3] = -float(np.dot(n, c))
    f[4:7] = c
    w = f.view(np.int32).copy()
    w[7], w[8], w[9], w[10] = inliers, inliers, 0, status
    return w


def _table(rows):
    return torch.from_numpy(np.stack(rows))


def _frame_dicts(table):
    t = table.numpy()
    f = t.view(np.float32)
    return [{"n": [float(v) for v in f[i, 0:3]], "c": [float(v) for v in f[i, 4:7]], "inliers": int(t[i, 7]),
             "status": int(t[i, 10])} for i in range(t.shape[0])]


IDENT = [1.0, 0, 0, 0, 0, 1.0, 0, 0, 0, 0, 1.0, 0, 0, 0, 0, 1.0]


# ------------------------------------------------------------------ Eqs. 6-10
def test_kalman_worked_example():
    # x=0, P=1, sigma_p=0, sigma_m=1, z=0.01 -> K=0.5, x=0.005, P=0.5
    x, P, K = orc.kalman_step(0.0, 1.0, 0.01, 0.0, 1.0)
    assert (K, x, P) == (0.5, 0.005, 0.5)
    f = pm.pm_drift_filter(0.0, 1.0)
    K2 = pm.drift_kalman_step(f, 0.01, 0.0, 1.0)
    assert (K2, f.x, f.P) == (0.5, 0.005, 0.5)


def test_kalman_limits_and_convergence():
    # sigma_m -> large: the measurement is ignored
    f = pm.pm_drift_filter(0.0, 1.0)
    pm.drift_kalman_step(f, 0.03, 0.0, 1e12)
    assert abs(f.x) < 1e-9
    # constant z repeated: x -> z
    f = pm.pm_drift_filter(0.0, 1.0)
    for _ in range(50):
        pm.drift_kalman_step(f, 0.03, 1e-6, 1e-4)
    assert 0.029 <= f.x <= 0.031
    # sigma_p = 0: P strictly positive and non-increasing
    f = pm.pm_drift_filter(0.0, 0.7)
    prev = f.P
    for k in range(100):
        pm.drift_kalman_step(f, 0.01 * math.sin(k), 0.0, 0.2)
        assert 0.0 < f.P <= prev
        prev = f.P


@pytest.mark.parametrize("sp,sm", [(1e-4, 1e-4), (1e-2, 1e-6), (1e-6, 1e-2), (0.3, 2.0)])
def test_kalman_steady_state_closed_form(sp, sm):
    # fixed point of Eqs. 7, 8, 10: Q = P + sp with P = Q sm / (Q + sm)
    #   => Q^2 - sp Q - sp sm = 0,  Q = (sp + sqrt(sp^2 + 4 sp sm)) / 2
    Q = (sp + math.sqrt(sp * sp + 4 * sp * sm)) / 2
    f = pm.pm_drift_filter(0.0, 1.0)
    for _ in range(20000):
        pm.drift_kalman_step(f, 0.0, sp, sm)
    assert math.isclose(f.P, Q - sp, rel_tol=1e-9)


def test_kalman_product_equals_oracle():
    rng = random.Random(3)
    f = pm.pm_drift_filter(0.01, 0.5)
    x, P = 0.01, 0.5
    for _ in range(500):
        z, sp, sm = rng.uniform(-0.1, 0.1), rng.uniform(0, 1e-2), rng.uniform(1e-6, 1e-1)
        K = pm.drift_kalman_step(f, z, sp, sm)
        x, P, K2 = orc.kalman_step(x, P, z, sp, sm)
        assert (f.x, f.P, K) == (x, P, K2)


# ------------------------------------------------------------------ Eqs. 4-5
def test_merge_gate():
    # Eq. 5 is "<=": exactly at the tolerance merges (dyadic values, exact dz)
    assert pm.merge_gate(0.5, 0.5625, 0.0625) == (0.0625, True)
    assert pm.merge_gate(0.5625, 0.5, 0.0625) == (0.0625, True)
    assert pm.merge_gate(0.5, 0.5625, 0.0625 - 2 ** -40)[1] is False
    # paper tolerance 5 cm: 6 cm apart -> no merge
    assert pm.merge_gate(1.0, 1.06, 0.05)[1] is False
    assert pm.merge_gate(1.0, 1.04, 0.05)[1] is True
    for a, b in [(0.3, 0.33), (2.0, 1.95), (-1.0, -1.0)]:
        assert pm.merge_gate(a, b, 0.05) == orc.merge_gate(a, b, 0.05)


# ------------------------------------------------------------------ map steps
def _pose(yaw=0.0, t=(0.0, 0.0, 0.0)):
    c, s = math.cos(yaw), math.sin(yaw)
    return [c, -s, 0, t[0], s, c, 0, t[1], 0, 0, 1, t[2], 0, 0, 0, 1]


def test_map_scenarios_from_spec():
    floor = _row([0, 0, 1], [0.2, 0.1, 0.0], inliers=1000)
    # empty map + one plane -> inserted, no drift update
    M = pm.PlaneMap(sigma_p=1.0, sigma_m=1e-6)
    match, zk = M.merge_frame(_table([floor]), IDENT)
    assert match == [-1] and zk is None and M.count.value == 1 and M.filter.x == 0.0
    # re-observed with +0.02 m vertical odometry error, sigma_p >> sigma_m:
    # merged, drift estimate ~0.02, stored z within 1 mm of the original
    match, zk = M.merge_frame(_table([floor]), _pose(t=(0, 0, 0.02)))
    assert match == [0] and abs(zk - 0.02) < 1e-9 and abs(M.filter.x - 0.02) < 1e-5
    assert M.count.value == 1 and abs(M.as_list()[0]["c"][2]) < 1e-3 and M.as_list()[0]["n_obs"] == 2
    # re-observation at dz = 0.08 m (beyond 5 cm) -> inserted separately
    M2 = pm.PlaneMap()
    M2.merge_frame(_table([floor]), IDENT)
    match, zk = M2.merge_frame(_table([floor]), _pose(t=(0, 0, 0.08)))
    assert match == [-1] and zk is None and M2.count.value == 2
    # rejected planes are ignored
    M3 = pm.PlaneMap()
    match, _ = M3.merge_frame(_table([_row([0, 0, 1], [0, 0, 0], status=1)]), IDENT)
    assert match == [-1] and M3.count.value == 0


def test_map_product_equals_oracle_random_sequences():
    rng = np.random.default_rng(11)
    params = {"drift_tol": 0.05, "normal_tol": 0.2, "xy_radius": 0.6, "sigma_p": 1e-3, "sigma_m": 1e-4}
    M = pm.PlaneMap(capacity=512, **params)
    omap, ox, oP = [], 0.0, 1.0
    # a static staircase of 6 treads and 5 risers seen from drifting poses
    treads = [([0, 0, 1], [0.3 * k, 0.0, 0.15 * k]) for k in range(6)]
    risers = [([1, 0, 0], [0.3 * k + 0.15, 0.0, 0.15 * k + 0.07]) for k in range(5)]
    drift = 0.0
    for frame in range(30):
        drift += rng.uniform(-0.004, 0.006)
        yaw = rng.uniform(-0.3, 0.3)
        pose = _pose(yaw, (rng.uniform(-0.1, 0.1), rng.uniform(-0.1, 0.1), drift))
        R = np.array(pose).reshape(4, 4)[:3, :3]
        t = np.array(pose).reshape(4, 4)[:3, 3]
        rows = []
        for n, c in treads + risers:
            if rng.random() < 0.3:
                continue
            # camera-frame observation of the world plane (noise ~ mm / 1 deg)
            nc = R.T @ np.array(n, float) + rng.normal(0, 0.01, 3)
            nc /= np.linalg.norm(nc)
            cc = R.T @ (np.array(c, float) + rng.normal(0, 0.003, 3) - t)
            rows.append(_row(nc, cc, inliers=int(rng.integers(300, 5000)), status=int(rng.random() < 0.1)))
        tab = _table(rows)
        match, zk = M.merge_frame(tab, pose)
        omap, ox, oP, omatch, ozk = orc.merge_frame(omap, _frame_dicts(tab), pose, ox, oP, params)
        assert match == omatch
        assert (zk is None) == (ozk is None) and (zk is None or abs(zk - ozk) <= 1e-12)
        assert abs(M.filter.x - ox) <= 1e-12 and abs(M.filter.P - oP) <= 1e-12
        got = M.as_list()
        assert len(got) == len(omap)
        for g, o in zip(got, omap):
            assert np.allclose(g["n"], o["n"], atol=1e-12) and np.allclose(g["c"], o["c"], atol=1e-12)
            assert g["w"] == o["w"] and g["n_obs"] == o["n_obs"]
    # the drift compensation keeps the map compact: one entry per physical plane
    assert len(omap) <= 2 * len(treads + risers)


def test_map_capacity_overflow_leaves_map_untouched():
    M = pm.PlaneMap(capacity=2)
    rows = [_row([0, 0, 1], [k, 0, 0.0]) for k in range(3)]
    with pytest.raises(pm.PMError):
        M.merge_frame(_table(rows), IDENT)
    assert M.count.value == 0 and M.filter.x == 0.0


# ------------------------------------------------------------------ oracle pins
# The checks below run on oracle/mapman.py ALONE (no product code), so a
# pose-convention mistake shared by the oracle and csrc/mapman.cpp fails here.
def test_oracle_to_world_closed_forms():
    # yaw +90 deg about world z (n_w = R n, c_w = R c + t; the pose
    # is the row-major 4x4 camera-to-world matrix): camera x -> world y,
    # camera y -> world -x, camera z -> world z
    P = _pose(math.pi / 2, (10.0, 20.0, 30.0))
    nw, cw = orc.to_world([1.0, 0.0, 0.0], [1.0, 2.0, 3.0], P)
    assert np.allclose(nw, [0.0, 1.0, 0.0], atol=1e-15)
    assert np.allclose(cw, [10.0 - 2.0, 20.0 + 1.0, 30.0 + 3.0], atol=1e-12)
    nw, _ = orc.to_world([0.0, 1.0, 0.0], [0.0, 0.0, 0.0], P)
    assert np.allclose(nw, [-1.0, 0.0, 0.0], atol=1e-15)
    # pitch -90 deg about world x (rows of R: (1,0,0), (0,0,1), (0,-1,0)): a
    # camera looking along its +z sees the floor normal (0,-1,0)... maps to +z up
    Px = [1, 0, 0, 0.5, 0, 0, 1, 0.0, 0, -1, 0, 2.0, 0, 0, 0, 1]
    nw, cw = orc.to_world([0.0, -1.0, 0.0], [0.0, 0.0, 1.5], Px)
    assert np.allclose(nw, [0.0, 0.0, 1.0]) and np.allclose(cw, [0.5, 1.5, 2.0])
    # the translation is the last column (indices 3, 7, 11), not the last row
    nw, cw = orc.to_world([0.0, 0.0, 1.0], [0.0, 0.0, 0.0], [1, 0, 0, 4, 0, 1, 0, 5, 0, 0, 1, 6, 7, 8, 9, 1])
    assert cw == [4.0, 5.0, 6.0] and nw == [0.0, 0.0, 1.0]


def _oplane(n, c, inliers=100, status=0):
    return {"n": list(map(float, n)), "c": list(map(float, c)), "inliers": inliers, "status": status}


def test_oracle_map_scenarios_from_spec():
    prm = {"drift_tol": 0.05, "normal_tol": math.radians(10), "xy_radius": 0.5, "sigma_p": 1.0, "sigma_m": 1e-6}
    floor = _oplane([0, 0, 1], [0.2, 0.1, 0.0], inliers=1000)
    # empty map + one plane -> one entry, no drift update
    m, x, P, match, zk = orc.merge_frame([], [floor], IDENT, 0.0, 1.0, prm)
    assert match == [-1] and zk is None and len(m) == 1 and (x, P) == (0.0, 1.0)
    assert m[0]["c"] == [0.2, 0.1, 0.0] and m[0]["w"] == 1000.0 and m[0]["n_obs"] == 1
    # the same plane re-observed with +2 cm vertical odometry error,
    # sigma_p >> sigma_m -> merged, z_k = 0.02, x -> 0.02, the stored height
    # stays within 1 mm of the original
    m2, x2, P2, match, zk = orc.merge_frame(m, [floor], _pose(t=(0, 0, 0.02)), x, P, prm)
    assert match == [0] and abs(zk - 0.02) < 1e-12 and abs(x2 - 0.02) < 1e-5
    assert len(m2) == 1 and abs(m2[0]["c"][2]) < 1e-3 and m2[0]["n_obs"] == 2 and m2[0]["w"] == 2000.0
    # dz = 8 cm > 5 cm -> inserted as a separate entry, no drift update
    m3, x3, _, match, zk = orc.merge_frame(m, [floor], _pose(t=(0, 0, 0.08)), 0.0, 1.0, prm)
    assert match == [-1] and zk is None and len(m3) == 2 and x3 == 0.0
    assert abs(m3[1]["c"][2] - 0.08) < 1e-12
    # 49 mm merges, 51 mm inserts (Eq. 5 with the 5 cm tolerance)
    for dz, merged in [(0.049, True), (0.051, False)]:
        _, _, _, match, _ = orc.merge_frame(m, [floor], _pose(t=(0, 0, dz)), 0.0, 1.0, prm)
        assert (match == [0]) is merged
    # rejected planes (status != OK) never enter the map
    m4, _, _, match, _ = orc.merge_frame([], [_oplane([0, 0, 1], [0, 0, 0], status=1)], IDENT, 0.0, 1.0, prm)
    assert match == [-1] and m4 == []
    # the gate is on normals: a wall at the same height is not merged into the floor
    wall = _oplane([1, 0, 0], [0.2, 0.1, 0.0])
    m5, _, _, match, _ = orc.merge_frame(m, [wall], IDENT, 0.0, 1.0, prm)
    assert match == [-1] and len(m5) == 2


def _stair_world(steps=5):
    return [([0.0, 0.0, 1.0], [0.3 * k + 0.15, 0.0, -0.15 * k]) for k in range(steps)]


def _observe(treads, yaw, t_true):
    """Camera-frame planes of world treads seen from the true pose (R, t_true)."""
    R = np.array(_pose(yaw, t_true)).reshape(4, 4)[:3, :3]
    t = np.array(t_true, float)
    return [_oplane(R.T @ np.array(n), R.T @ (np.array(c) - t), inliers=2000) for n, c in treads]


def _drift_run(compensate):
    # SPEC acceptance 5: linear vertical drift of 2 mm per frame over
    # 50 frames; the odometry pose is the true pose shifted up by the drift
    treads = _stair_world()
    prm = {"drift_tol": 0.05, "normal_tol": math.radians(10), "xy_radius": 0.5,
           "sigma_p": 1.0 if compensate else 0.0, "sigma_m": 1e-6 if compensate else 1e12}
    m, x, P = [], 0.0, 1e-6
    for k in range(50):
        yaw = 0.2 * math.sin(0.3 * k)
        t_true = (0.05 * k, 0.01 * k, 1.2)
        drift = 0.002 * k
        pose = _pose(yaw, (t_true[0], t_true[1], t_true[2] + drift))
        m, x, P, _, _ = orc.merge_frame(m, _observe(treads, yaw, t_true), pose, x, P, prm)
    err = max(min(abs(e["c"][2] - c[2]) for _, c in treads) for e in m)
    return m, x, err


def test_oracle_drift_tracking_acceptance():
    m, x, err = _drift_run(True)
    injected = 0.002 * 49
    assert abs(x - injected) <= 0.2 * injected          # final x-hat within 20 %
    assert err <= 0.005                                 # every tread centroid within 5 mm of truth
    assert len(m) == 5                                  # one entry per tread
    # without compensation (filter frozen) the heights spread beyond 50 mm
    m0, x0, err0 = _drift_run(False)
    assert abs(x0) < 1e-9 and err0 > 0.05 and len(m0) > 5
