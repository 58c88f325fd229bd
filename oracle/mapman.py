"""Oracle for NEXT-4: the paper's map merge gate (Eqs. 4-5)
and scalar vertical-drift Kalman filter (Eqs. 6-10), applied to the plane
table the hot path outputs (one plane per region instead of a polygon, DESIGN.md
readings Q30-Q34).  TEST INFRASTRUCTURE ONLY: imported by tests/ alone; the
product implementation is the library's host code (csrc/mapman.cpp,
pm_drift_kalman_step / pm_merge_gate / pm_plane_map_merge_frame).

Plain Python, fp64, one statement per equation in the paper's order.
Citations: PAPER.md lines (P:nnn), SPEC.md lines (S:nnn)."""
import math


def kalman_step(x, P, z, sigma_p, sigma_m):
    """Eqs. 6-10, in order.  Returns (x_k|k, P_k|k, K_k)."""
    x_pred = x                                  # Eq. 6: x_k|k-1 = x_k-1|k-1
    P_pred = P + sigma_p                        # Eq. 7: P_k|k-1 = P_k-1|k-1 + sigma_p
    K = P_pred / (P_pred + sigma_m)             # Eq. 8
    x_new = x_pred + K * (z - x_pred)           # Eq. 9
    P_new = (1.0 - K) * P_pred                  # Eq. 10
    return x_new, P_new, K


def merge_gate(z_new, z_map, drift_tol):
    """Eqs. 4-5: dz = |z_new - z|, merge iff dz <= tolerance."""
    dz = abs(z_new - z_map)                     # Eq. 4
    return dz, dz <= drift_tol                  # Eq. 5


def to_world(n, c, pose):
    """Rigid transform of a camera-frame plane (normal n, centroid c) by the
    4x4 camera-to-world pose: n_w = R n, c_w = R c + t."""
    R = [[pose[4 * i + j] for j in range(3)] for i in range(3)]
    t = [pose[3], pose[7], pose[11]]
    nw = [sum(R[i][j] * n[j] for j in range(3)) for i in range(3)]
    cw = [sum(R[i][j] * c[j] for j in range(3)) + t[i] for i in range(3)]
    return nw, cw


def _angle(a, b):
    d = sum(a[i] * b[i] for i in range(3))
    na = math.sqrt(sum(v * v for v in a))
    nb = math.sqrt(sum(v * v for v in b))
    return math.acos(max(-1.0, min(1.0, abs(d) / (na * nb))))


def merge_frame(map_planes, frame, pose, x, P, params):
    """One frame into the plane map (S:426-430 pipeline, planes for polygons):
      (1) to_world every OK plane; (2) z -= x (current drift estimate);
      (3) match each incoming plane to the map plane that passes the gate
          (normals within normal_tol, horizontal centroid distance <= xy_radius,
          Eq. 5 on the centroid heights) with the smallest horizontal distance
          (ties -> lowest map index);
      (4) if any matched: z_k = mean signed (z_new - z_map) + x,
          Kalman step (Eqs. 6-10), incoming z -= (x_new - x_old);
      (5) matched pairs merged: weights = inlier counts, n = normalised
          weighted sum (oriented like the map plane), c = weighted mean;
          unmatched planes inserted (in frame order).
    map_planes: list of dicts {n, c, w, n_obs}; frame: list of dicts
    {n, c, inliers, status}.  Returns (map, x, P, matches, z_k or None)."""
    tol, ntol, rxy = params["drift_tol"], params["normal_tol"], params["xy_radius"]
    inc = []
    for f in frame:
        if f["status"] != 0:
            inc.append(None)
            continue
        nw, cw = to_world(f["n"], f["c"], pose)
        cw[2] -= x
        inc.append({"n": nw, "c": cw, "w": float(f["inliers"])})
    match = [-1] * len(frame)
    resid = []
    for i, p in enumerate(inc):
        if p is None:
            continue
        best, bd = -1, None
        for j, m in enumerate(map_planes):
            if _angle(p["n"], m["n"]) > ntol:
                continue
            dxy = math.hypot(p["c"][0] - m["c"][0], p["c"][1] - m["c"][1])
            if dxy > rxy:
                continue
            _, ok = merge_gate(p["c"][2], m["c"][2], tol)
            if not ok:
                continue
            if bd is None or dxy < bd:
                best, bd = j, dxy
        match[i] = best
        if best >= 0:
            resid.append(p["c"][2] - map_planes[best]["c"][2])
    zk = None
    if resid:
        zk = sum(resid) / len(resid) + x
        x_old = x
        x, P, _ = kalman_step(x, P, zk, params["sigma_p"], params["sigma_m"])
        for p in inc:
            if p is not None:
                p["c"][2] -= (x - x_old)
    out = [dict(m) for m in map_planes]
    for i, p in enumerate(inc):
        if p is None:
            continue
        j = match[i]
        if j < 0:
            out.append({"n": p["n"], "c": p["c"], "w": p["w"], "n_obs": 1})
            continue
        m = out[j]
        s = 1.0 if sum(p["n"][k] * m["n"][k] for k in range(3)) >= 0 else -1.0
        wa, wb = m["w"], p["w"]
        nn = [wa * m["n"][k] + wb * s * p["n"][k] for k in range(3)]
        L = math.sqrt(sum(v * v for v in nn))
        out[j] = {"n": [v / L for v in nn], "c": [(wa * m["c"][k] + wb * p["c"][k]) / (wa + wb) for k in range(3)],
                  "w": wa + wb, "n_obs": m["n_obs"] + 1}
    return out, x, P, match, zk
