"""Seeded synthetic depth-frame generators (shared test/bench INPUT module).

This module only produces inputs: depth frames (float32 metres, 0 = invalid)
with the structure of the paper's workloads (descending straight and spiral
staircases seen by a ground-pointing depth camera, P:24 ``fig:p0``, P:126;
320x240 / 640x480 frames), region-label images, camera
intrinsics and ground-truth planes.  It holds none of the method's arithmetic
(no diffusion, no normals, no RANSAC) and is imported by both the oracle tests
and the CUDA path's tests / bench.  Recipes: DESIGN.md §4 (after SURVEY
§8(d)).  All randomness comes from an integer hash of (seed, frame, pixel) or
from a seeded ``torch.Generator`` — never from global RNG state.

Geometry is computed in float64 with torch, on any device; the frame is
rounded to float32 at the end.
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import torch

__all__ = [
    "Intrinsics", "intrinsics_for", "stair", "ramp", "spiral", "terrain",
    "d435_noise", "l515_noise", "dropout", "balanced_labels", "make_config",
    "stair_stream", "CONFIGS", "DEFAULTS",
]

# Library / config defaults (DESIGN.md §3 readings Q5, Q16): lambda=gamma,
# kappa=k in metres, tau in metres, RANSAC seed.
DEFAULTS = dict(lam=0.15, kappa=0.03, tau=0.01, seed=0x1919)


@dataclass(frozen=True)
class Intrinsics:
    """Pinhole intrinsics (Q24): u = column, v = row, pixel centres at integers."""
    fx: float
    fy: float
    cx: float
    cy: float


def intrinsics_for(W: int, H: int) -> Intrinsics:
    """§8(d): fx = fy = 385 W/640 for 4:3 frames; 1280x720 -> 640;
    4096x3072 -> 2048; principal point ((W-1)/2, (H-1)/2)."""
    if (W, H) == (1280, 720):
        f = 640.0
    elif (W, H) == (4096, 3072):
        f = 2048.0
    else:
        f = 385.0 * W / 640.0
    return Intrinsics(f, f, (W - 1) / 2.0, (H - 1) / 2.0)


# --------------------------------------------------------------------------
# integer hash (Wellons "lowbias32") on int64 tensors; all products < 2^63
_M32 = 0xFFFFFFFF


def _hash32(x: torch.Tensor) -> torch.Tensor:
    x = x & _M32
    x = x ^ (x >> 16)
    x = (x * 0x7FEB352D) & _M32
    x = x ^ (x >> 15)
    x = (x * 0x846CA68B) & _M32
    x = x ^ (x >> 16)
    return x


def _uniform(seed: int, frame: int, stream: int, n: int, device) -> torch.Tensor:
    """n uniforms in (0, 1), float64, keyed on (seed, frame, stream, index)."""
    i = torch.arange(n, device=device, dtype=torch.int64)
    h = _hash32(i ^ _hash32(torch.full_like(i, (seed * 0x9E3779B1 + frame * 0x85EBCA77 + stream * 0xC2B2AE3D) & _M32)))
    h = _hash32(h + i * 0x27D4EB2F)
    return (h.to(torch.float64) + 0.5) / 4294967296.0


def _gauss(seed: int, frame: int, n: int, device) -> torch.Tensor:
    u1 = _uniform(seed, frame, 1, n, device)
    u2 = _uniform(seed, frame, 2, n, device)
    return torch.sqrt(-2.0 * torch.log(u1)) * torch.cos(2.0 * math.pi * u2)


def _rays(W: int, H: int, K: Intrinsics, device):
    v, u = torch.meshgrid(torch.arange(H, device=device, dtype=torch.float64),
                          torch.arange(W, device=device, dtype=torch.float64), indexing="ij")
    return (u - K.cx) / K.fx, (v - K.cy) / K.fy


def _camera_axes(pitch_deg: float, yaw_deg: float):
    """World z up.  Camera frame x right, y down (image rows), z forward;
    forward pitched `pitch` below the horizon, heading rotated by `yaw`
    about world z (yaw 0 looks along +y)."""
    p, y = math.radians(pitch_deg), math.radians(yaw_deg)
    h = (math.sin(y), math.cos(y), 0.0)
    f = (math.cos(p) * h[0], math.cos(p) * h[1], -math.sin(p))
    xc = (math.cos(y), -math.sin(y), 0.0)
    yc = (f[1] * xc[2] - f[2] * xc[1], f[2] * xc[0] - f[0] * xc[2], f[0] * xc[1] - f[1] * xc[0])
    return xc, yc, f


def _world_rays(W, H, K, pitch_deg, yaw_deg, device):
    a, b = _rays(W, H, K, device)
    xc, yc, f = _camera_axes(pitch_deg, yaw_deg)
    r = [a * xc[i] + b * yc[i] + f[i] for i in range(3)]
    return r, (xc, yc, f)


def _plane_cam(n_w, d_w, axes, cam):
    """World plane n.X + d = 0 -> camera frame (n_c, d_c), oriented d_c >= 0."""
    xc, yc, f = axes
    n_c = [sum(n_w[i] * ax[i] for i in range(3)) for ax in (xc, yc, f)]
    d_c = d_w + sum(n_w[i] * cam[i] for i in range(3))
    if d_c < 0:
        n_c, d_c = [-x for x in n_c], -d_c
    return (tuple(n_c), d_c)


# --------------------------------------------------------------------------
def stair(W: int, H: int, K: Intrinsics, steps: int = 3, pitch_deg: float = 55.0,
          height: float = 0.8, yaw_deg: float = 0.0, rise: float = 0.15, run: float = 0.28,
          nosing: float = 0.6, device="cpu"):
    """G-STAIR (descending view, §8(d)): camera `height` above the top
    landing (world z = 0), pitched down; tread k (k = 1..steps) is the
    horizontal plane z = -rise k for y in [nosing + run (k-1), nosing + run k);
    the last one extends to infinity; risers face away (invisible).
    Returns (depth float64 [H, W] with 0 = miss, face id int32 [H, W] with -1 =
    miss, ground-truth camera-frame planes [(n, d)] per face)."""
    r, axes = _world_rays(W, H, K, pitch_deg, yaw_deg, device)
    cam = (0.0, 0.0, height)
    depth = torch.zeros(H, W, dtype=torch.float64, device=device)
    face = torch.full((H, W), -1, dtype=torch.int32, device=device)
    down = r[2] < 0
    planes = []
    for k in range(steps + 1):
        zk = -rise * k
        t = (zk - height) / torch.where(down, r[2], torch.full_like(r[2], -1.0))
        y = cam[1] + t * r[1]
        lo = -math.inf if k == 0 else nosing + run * (k - 1)
        hi = math.inf if k == steps else nosing + run * k
        hit = down & (face < 0) & (y >= lo) & (y < hi) & (t > 0)
        depth = torch.where(hit, t, depth)
        face = torch.where(hit, torch.full_like(face, k), face)
        planes.append(_plane_cam((0.0, 0.0, 1.0), -zk, axes, cam))
    return depth, face, planes


def ramp(W: int, H: int, K: Intrinsics, tilt_deg: float = 30.0, azim_deg: float = 35.0,
         d: float = 1.5, device="cpu"):
    """G-RAMP: one analytic plane n.X + d = 0 in the camera frame, its normal
    `tilt` off the optical axis (facing the camera), distance d.  Depth
    z = -d / (n . (a, b, 1)).  Returns (depth, face, [(n, d)])."""
    t, az = math.radians(tilt_deg), math.radians(azim_deg)
    n = (math.sin(t) * math.cos(az), math.sin(t) * math.sin(az), -math.cos(t))
    a, b = _rays(W, H, K, device)
    den = n[0] * a + n[1] * b + n[2]
    ok = den < 0
    depth = torch.where(ok, -d / torch.where(ok, den, torch.full_like(den, -1.0)), torch.zeros_like(den))
    face = torch.where(ok, 0, -1).to(torch.int32)
    return depth, face, [(n, d)]


def spiral(W: int, H: int, K: Intrinsics, n_treads: int = 16, sector_deg: float = 22.5,
           r_in: float = 0.15, r_out: float = 1.0, rise: float = 0.18, cam_radius: float = 1.6,
           cam_above: float = 0.8, pitch_deg: float = 65.0, device="cpu"):
    """G-SPIRAL (§8(d)): n_treads horizontal annular-sector treads (inner
    r_in, outer r_out, sector_deg each) descending counter-clockwise around
    the world z axis, tread k at z = rise (n_treads - k); a floor at z = 0 and
    a solid central column r < r_in up to the top tread (valid depth, face -1
    in the label sense: returned face id = -2).  Camera cam_above over the top
    tread at radius cam_radius on the +x axis, pitched toward the axis.
    Faces: 0..n_treads-1 treads, n_treads = floor."""
    z_top = rise * n_treads
    cz = z_top + cam_above
    cam = (cam_radius, 0.0, cz)
    # heading toward the axis = -x  <=> yaw = -90 deg in our convention
    r, axes = _world_rays(W, H, K, pitch_deg, -90.0, device)
    inf = torch.full_like(r[0], math.inf)
    best_t = inf.clone()
    face = torch.full((H, W), -1, dtype=torch.int32, device=device)
    sec = math.radians(sector_deg)
    rz = torch.where(r[2] < 0, r[2], torch.full_like(r[2], -1e-300))
    planes = []
    for k in range(n_treads + 1):
        zk = rise * (n_treads - k) if k < n_treads else 0.0
        t = (zk - cz) / rz
        x = cam[0] + t * r[0]
        y = cam[1] + t * r[1]
        ok = (r[2] < 0) & (t > 0)
        if k < n_treads:
            rad = torch.sqrt(x * x + y * y)
            ang = torch.remainder(torch.atan2(y, x) + sec / 2.0, 2 * math.pi)
            ok = ok & (rad >= r_in) & (rad < r_out) & (ang >= k * sec) & (ang < (k + 1) * sec)
        upd = ok & (t < best_t)
        best_t = torch.where(upd, t, best_t)
        face = torch.where(upd, torch.full_like(face, k), face)
        planes.append(_plane_cam((0.0, 0.0, 1.0), -zk, axes, cam))
    # column: side  (x^2 + y^2 = r_in^2, 0 <= z <= z_top) and top cap
    A = r[0] * r[0] + r[1] * r[1]
    B = 2.0 * (cam[0] * r[0] + cam[1] * r[1])
    C = cam[0] ** 2 + cam[1] ** 2 - r_in ** 2
    disc = B * B - 4 * A * C
    okd = disc >= 0
    t_side = (-B - torch.sqrt(torch.clamp(disc, min=0.0))) / (2 * A)
    z_side = cz + t_side * r[2]
    ok_side = okd & (t_side > 0) & (z_side >= 0) & (z_side <= z_top) & (t_side < best_t)
    best_t = torch.where(ok_side, t_side, best_t)
    face = torch.where(ok_side, torch.full_like(face, -2), face)
    t_cap = (z_top - cz) / rz
    xc_, yc_ = cam[0] + t_cap * r[0], cam[1] + t_cap * r[1]
    ok_cap = (r[2] < 0) & (t_cap > 0) & (xc_ * xc_ + yc_ * yc_ < r_in ** 2) & (t_cap < best_t)
    best_t = torch.where(ok_cap, t_cap, best_t)
    face = torch.where(ok_cap, torch.full_like(face, -2), face)
    depth = torch.where(torch.isfinite(best_t), best_t, torch.zeros_like(best_t))
    return depth, face, planes


def terrain(W: int, H: int, K: Intrinsics, grid: int = 32, seed: int = 5, max_tilt_deg: float = 30.0,
            zmin: float = 1.5, zmax: float = 3.0, device="cpu"):
    """G-TERRAIN (§8(d)): grid x grid facets in image space; facet (i, j) is
    an analytic plane whose depth on its centre ray is U[zmin, zmax] and whose
    normal is within max_tilt of that ray, reversed to face the camera.
    Face id = i * grid + j."""
    g = torch.Generator(device="cpu").manual_seed(seed)
    nf = grid * grid
    zc = zmin + (zmax - zmin) * torch.rand(nf, generator=g, dtype=torch.float64)
    cos_t = 1 - torch.rand(nf, generator=g, dtype=torch.float64) * (1 - math.cos(math.radians(max_tilt_deg)))
    phi = 2 * math.pi * torch.rand(nf, generator=g, dtype=torch.float64)
    fw, fh = W / grid, H / grid
    jj = torch.arange(nf) % grid
    ii = torch.arange(nf) // grid
    uc = (jj.to(torch.float64) + 0.5) * fw - 0.5
    vc = (ii.to(torch.float64) + 0.5) * fh - 0.5
    ray = torch.stack([(uc - K.cx) / K.fx, (vc - K.cy) / K.fy, torch.ones(nf, dtype=torch.float64)], 1)
    w = -ray / ray.norm(dim=1, keepdim=True)            # toward the camera
    # orthonormal frame around w
    tmp = torch.where((w[:, 0].abs() < 0.9).unsqueeze(1), torch.tensor([1.0, 0, 0], dtype=torch.float64),
                      torch.tensor([0, 1.0, 0], dtype=torch.float64))
    e1 = torch.linalg.cross(w, tmp)
    e1 = e1 / e1.norm(dim=1, keepdim=True)
    e2 = torch.linalg.cross(w, e1)
    sin_t = torch.sqrt(1 - cos_t ** 2)
    n = cos_t[:, None] * w + sin_t[:, None] * (torch.cos(phi)[:, None] * e1 + torch.sin(phi)[:, None] * e2)
    P = zc[:, None] * ray
    d = -(n * P).sum(1)                                   # n.P + d = 0 ; d > 0 since n faces camera
    a, b = _rays(W, H, K, device)
    v, u = torch.meshgrid(torch.arange(H, device=device), torch.arange(W, device=device), indexing="ij")
    fi = torch.clamp((v.to(torch.float64) / fh).floor().long(), max=grid - 1)
    fj = torch.clamp((u.to(torch.float64) / fw).floor().long(), max=grid - 1)
    fid = fi * grid + fj
    nd = n.to(device)[fid]
    dd = d.to(device)[fid]
    den = nd[..., 0] * a + nd[..., 1] * b + nd[..., 2]
    depth = -dd / den
    planes = [(tuple(n[k].tolist()), float(d[k])) for k in range(nf)]
    return depth, fid.to(torch.int32), planes


# --------------------------------------------------------------------------
def d435_noise(depth: torch.Tensor, K: Intrinsics, seed: int, frame: int = 0,
               subpixel: float = 0.08, baseline: float = 0.05) -> torch.Tensor:
    """D435-style stereo noise (§8(d)): z' = round_mm(z + sigma(z) xi),
    sigma(z) = subpixel z^2 / (fx baseline); xi ~ N(0, 1) from the hash.
    Invalid (0) stays 0.  float64 in, float64 out (mm-quantised)."""
    xi = _gauss(seed, frame, depth.numel(), depth.device).view_as(depth)
    sigma = subpixel * depth * depth / (K.fx * baseline)
    z = torch.round((depth + sigma * xi) * 1000.0) / 1000.0
    return torch.where(depth > 0, torch.clamp(z, min=1e-3), depth)


def l515_noise(depth: torch.Tensor, seed: int, frame: int = 0, sigma: float = 0.002) -> torch.Tensor:
    """L515-like noise for the terrain (§8(d)): sigma = 2 mm + 1 mm quantisation."""
    xi = _gauss(seed, frame, depth.numel(), depth.device).view_as(depth)
    z = torch.round((depth + sigma * xi) * 1000.0) / 1000.0
    return torch.where(depth > 0, torch.clamp(z, min=1e-3), depth)


def dropout(depth: torch.Tensor, rate: float, seed: int, frame: int = 0) -> torch.Tensor:
    """Set a `rate` fraction of pixels to 0 (invalid), hash-selected."""
    u = _uniform(seed, frame, 3, depth.numel(), depth.device).view_as(depth)
    return torch.where(u < rate, torch.zeros_like(depth), depth)


def balanced_labels(face: torch.Tensor, n_regions: int) -> torch.Tensor:
    """Balanced subdivision of ground-truth faces into exactly n_regions
    regions (§8(d)): region counts allocated to faces in proportion to pixel
    count (largest remainder); each face's raster-ordered pixel list split
    into that many contiguous chunks.  Guard: every region spans >= 3 rows and
    >= 3 columns, otherwise its face gets one region fewer (moved to the
    largest face).  Pixels with face < 0 get label -1."""
    H, W = face.shape
    dev = face.device
    flat = face.reshape(-1).long()
    valid = flat >= 0
    n_faces = int(flat.max().item()) + 1 if bool(valid.any()) else 0
    if n_faces == 0 or n_regions == 0:
        return torch.full_like(face, -1)
    counts = torch.bincount(flat[valid], minlength=n_faces).double().cpu()
    tot = counts.sum()
    quota_f = counts * n_regions / tot
    quota = quota_f.floor().long()
    rem = n_regions - int(quota.sum())
    order = torch.argsort(quota_f - quota.double(), descending=True, stable=True)
    quota[order[:rem]] += 1
    idx = torch.arange(flat.numel(), device=dev)
    rows, cols = idx // W, idx % W
    key = torch.where(valid, flat, torch.full_like(flat, n_faces))
    _, perm = torch.sort(key, stable=True)
    sorted_face = key[perm]
    starts = torch.zeros(n_faces + 2, dtype=torch.long, device=dev)
    starts[1:] = torch.cumsum(torch.bincount(sorted_face, minlength=n_faces + 1), 0)
    rank_sorted = torch.arange(flat.numel(), device=dev) - starts[sorted_face]
    rank = torch.empty_like(rank_sorted)
    rank[perm] = rank_sorted
    for _ in range(4 * n_regions + 8):
        q = quota.to(dev)
        base = torch.zeros(n_faces + 1, dtype=torch.long, device=dev)
        base[1:] = torch.cumsum(q, 0)
        cnt = counts.to(dev).long()
        fc = flat.clamp(min=0)
        local = torch.where(q[fc] > 0, (rank * q[fc]) // cnt[fc].clamp(min=1), torch.zeros_like(rank))
        lab = torch.where(valid & (q[fc] > 0), base[fc] + local, torch.full_like(flat, -1))
        lv = lab >= 0
        R = n_regions
        big = torch.full((R,), -1, dtype=torch.long, device=dev)
        small = torch.full((R,), 1 << 40, dtype=torch.long, device=dev)
        rmax = big.scatter_reduce(0, lab[lv], rows[lv], "amax")
        rmin = small.scatter_reduce(0, lab[lv], rows[lv], "amin")
        cmax = big.scatter_reduce(0, lab[lv], cols[lv], "amax")
        cmin = small.scatter_reduce(0, lab[lv], cols[lv], "amin")
        bad = ((rmax - rmin) < 2) | ((cmax - cmin) < 2)
        if not bool(bad.any()):
            break
        r_bad = int(torch.nonzero(bad)[0].item())
        f_bad = int(torch.searchsorted(base[1:].cpu(), torch.tensor(r_bad), right=True).item())
        quota[f_bad] -= 1
        quota[int(torch.argmax(counts).item())] += 1
    return lab.view(H, W).to(torch.int32)


# --------------------------------------------------------------------------
# BASELINE.json configs (§8(d) table)
CONFIGS = {
    "C1": dict(kind="stair", W=64, H=48, iters=10, n_regions=4, n_hyp=64, noise=False),
    "C1n": dict(kind="stair", W=64, H=48, iters=10, n_regions=4, n_hyp=64, noise=True),
    "C2": dict(kind="stair", W=640, H=480, iters=20, n_regions=32, n_hyp=64, noise=True),
    "C3": dict(kind="spiral", W=1280, H=720, iters=50, n_regions=128, n_hyp=256, noise=True),
    "C4": dict(kind="stair", W=640, H=480, iters=20, n_regions=64, n_hyp=64, noise=True),
    "C5": dict(kind="terrain", W=4096, H=3072, iters=100, n_regions=1024, n_hyp=64, noise=True),
    "RAMP": dict(kind="ramp", W=640, H=480, iters=0, n_regions=1, n_hyp=64, noise=False),
}


def make_config(name: str, W: int = None, H: int = None, holes: float = 0.0, noise=None,
                frame: int = 0, device="cpu") -> dict:
    """One frame of a BASELINE.json config (§8(d)); W/H override the size.
    Returns dict(depth=f32 [H,W] tensor, labels=int32 [H,W], K, planes, plus
    the config's iters / n_regions / n_hyp and the DEFAULTS)."""
    cfg = dict(CONFIGS[name])
    W = W or cfg["W"]
    H = H or cfg["H"]
    K = intrinsics_for(W, H)
    noise = cfg["noise"] if noise is None else noise
    seed = list(CONFIGS).index(name) + 1
    if cfg["kind"] == "stair":
        depth, face, planes = stair(W, H, K, device=device)
        if noise:
            depth = d435_noise(depth, K, seed, frame)
    elif cfg["kind"] == "spiral":
        depth, face, planes = spiral(W, H, K, device=device)
        if noise:
            depth = d435_noise(depth, K, seed, frame)
    elif cfg["kind"] == "terrain":
        depth, face, planes = terrain(W, H, K, device=device)
        if noise:
            depth = l515_noise(depth, seed, frame)
    elif cfg["kind"] == "ramp":
        depth, face, planes = ramp(W, H, K, device=device)
    else:
        raise ValueError(cfg["kind"])
    if holes > 0:
        depth = dropout(depth, holes, seed + 100, frame)
    if cfg["kind"] == "terrain" and cfg["n_regions"] == 1024 and (W, H) == (4096, 3072):
        labels = face.clone()
    elif cfg["kind"] == "stair" and cfg["n_regions"] == 4 and face.max() == 3:
        labels = face.clone()
    else:
        labels = balanced_labels(face, cfg["n_regions"])
    return dict(depth=depth.to(torch.float32), labels=labels.to(torch.int32), K=K, planes=planes,
                face=face, W=W, H=H, iters=cfg["iters"], n_regions=cfg["n_regions"],
                n_hyp=cfg["n_hyp"], **DEFAULTS)


def stair_params(frame: int) -> dict:
    """Per-frame pose of the C4 stream (§8(d)): pitch 50-60 deg, height
    0.8 +- 0.05 m, yaw +-10 deg, 3-5 steps, all from the frame index."""
    u = _uniform(0xC4, frame, 7, 4, "cpu").tolist()
    return dict(pitch_deg=50.0 + 10.0 * u[0], height=0.75 + 0.1 * u[1],
                yaw_deg=-10.0 + 20.0 * u[2], steps=3 + min(int(u[3] * 3), 2))


def stair_stream(first_frame: int, n_frames: int, W: int = 640, H: int = 480, n_regions: int = 64,
                 device="cpu"):
    """Frames [first_frame, first_frame + n_frames) of the C4 stream of
    distinct noisy G-STAIR frames.  Returns (depth f32 [B,H,W], labels int32
    [B,H,W], K).  Noise seed = frame index."""
    K = intrinsics_for(W, H)
    depth = torch.empty(n_frames, H, W, dtype=torch.float32, device=device)
    labels = torch.empty(n_frames, H, W, dtype=torch.int32, device=device)
    for i in range(n_frames):
        f = first_frame + i
        d, face, _ = stair(W, H, K, device=device, **stair_params(f))
        d = d435_noise(d, K, seed=f, frame=f)
        depth[i] = d.to(torch.float32)
        labels[i] = balanced_labels(face, n_regions)
    return depth, labels, K
