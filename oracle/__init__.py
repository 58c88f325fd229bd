"""ORACLE — test infrastructure only.

ctypes binding over ``oracle/oracle.c`` (plain single-threaded C; see its
header for what each function follows in arXiv 2411.01919).  Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py`` (its ``cpu_baseline`` leg and
``--impl reference``) may import this package.  The product path
(``paper_2411_01919_b200``) never imports it and shares no code with it.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB_PATH = os.path.join(_HERE, "liboracle.so")
_lock = threading.Lock()
_lib = None

CFLAGS = ["-O2", "-std=c11", "-fPIC", "-shared", "-ffp-contract=off", "-fno-fast-math",
          "-fvisibility=hidden", "-Wall", "-Wextra", "-Wno-unused-parameter"]

SAMPLER_PHILOX, SAMPLER_ENUMERATE = 0, 1
ADF_ALG1, ADF_DIVERGENCE = 0, 1
NORMALS_GEOMETRIC, NORMALS_AS_PRINTED = 0, 1
SELECT_COUNT, SELECT_ERROR, SELECT_COUNT_EARLY, SELECT_ERROR_EARLY = 0, 1, 2, 3
STATUS_OK, STATUS_REJECTED, STATUS_TOO_FEW, STATUS_DEGENERATE = 0, 1, 2, 3


def build(force: bool = False) -> str:
    """Compile liboracle.so with gcc (no FMA contraction)."""
    if force or not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(_SRC):
        tmp = _LIB_PATH + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", *CFLAGS, "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB_PATH)
    return _LIB_PATH


def lib() -> ctypes.CDLL:
    global _lib
    with _lock:
        if _lib is None:
            build()
            L = ctypes.CDLL(_LIB_PATH)
            P = ctypes.c_void_p
            i32, u32, u64, f32, f64 = (ctypes.c_int, ctypes.c_uint32, ctypes.c_uint64,
                                       ctypes.c_float, ctypes.c_double)
            L.orc_adf.argtypes = [P, P, i32, i32, f64, f64, i32]
            L.orc_adf_ex.argtypes = [P, P, i32, i32, f64, f64, i32, i32]
            L.orc_normals_ex.argtypes = [P, i32, i32, f64, f64, f64, f64, i32, P]
            L.orc_normals_f64_ex.argtypes = [P, i32, i32, f64, f64, f64, f64, i32, P]
            L.orc_normals.argtypes = [P, i32, i32, f64, f64, f64, f64, P]
            L.orc_normals_f64.argtypes = [P, i32, i32, f64, f64, f64, f64, P]
            L.orc_sobel_f64.argtypes = [P, i32, i32, P]
            L.orc_philox4x32_10.argtypes = [P, P, P]
            L.orc_philox4x32_10.restype = None
            L.orc_sample_triple.argtypes = [u32, u32, u32, u32, P]
            L.orc_sample_triple.restype = None
            L.orc_colex_unrank3.argtypes = [u64, u32, P]
            L.orc_deproject.argtypes = [i32, i32, f32, f32, f32, f32, f32, P]
            L.orc_deproject.restype = None
            L.orc_plane_from_3pts.argtypes = [P, P, P, P]
            L.orc_point_plane_dist.argtypes = [P, P]
            L.orc_point_plane_dist.restype = f32
            L.orc_refit_plane.argtypes = [P, i32, P]
            L.orc_ransac.argtypes = [P, P, i32, i32, f32, f32, f32, f32, i32, i32, f32, u64, u32,
                                     i32, i32, P, P, P, P, P]
            L.orc_normals_to_u8.argtypes = [P, i32, i32, P]
            L.orc_normals_to_u8.restype = None
            L.orc_canny_u8.argtypes = [P, i32, i32, i32, f64, f64, P]
            L.orc_segment_regions.argtypes = [P, i32, i32, f64, f64, i32, i32, P, P, P]
            L.orc_trace_contour.argtypes = [P, i32, i32, i32, P, i32]
            L.orc_simplify_dp.argtypes = [P, i32, i32, P]
            L.orc_rasterize_polygons.argtypes = [P, P, P, i32, i32, i32, P]
            L.orc_lift_vertices.argtypes = [P, i32, P, f64, f64, f64, f64, P]
            L.orc_lift_vertices.restype = None
            _lib = L
    return _lib


def _p(a: np.ndarray) -> int:
    return a.ctypes.data


def _c(a, dtype) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=dtype)


def adf(depth: np.ndarray, lam: float, kappa: float, iters: int, scheme: int = ADF_ALG1) -> np.ndarray:
    """Alg. 1 ℓ1-8 on one f32 [H, W] frame (metres) -> f32 [H, W].
    scheme=ADF_DIVERGENCE: Eq. 1 as the 4-flux Perona-Malik scheme."""
    d = _c(depth, np.float32)
    H, W = d.shape
    out = np.empty_like(d)
    rc = lib().orc_adf_ex(_p(d), _p(out), W, H, float(lam), float(kappa), int(iters), int(scheme))
    assert rc == 0
    return out


def normals(depth: np.ndarray, K, mode: int = NORMALS_GEOMETRIC) -> np.ndarray:
    """Alg. 1 ℓ9-13 on f32 depth -> float64 [3, H, W]; (0,0,0) = invalid.
    mode=NORMALS_AS_PRINTED: Eq. 2 literally."""
    d = _c(depth, np.float32)
    H, W = d.shape
    out = np.empty((3, H, W), np.float64)
    rc = lib().orc_normals_ex(_p(d), W, H, K.fx, K.fy, K.cx, K.cy, int(mode), _p(out))
    assert rc == 0
    return out


def normals_f64(depth: np.ndarray, K, mode: int = NORMALS_GEOMETRIC) -> np.ndarray:
    d = _c(depth, np.float64)
    H, W = d.shape
    out = np.empty((3, H, W), np.float64)
    rc = lib().orc_normals_f64_ex(_p(d), W, H, K.fx, K.fy, K.cx, K.cy, int(mode), _p(out))
    assert rc == 0
    return out


def sobel_f64(depth: np.ndarray) -> np.ndarray:
    d = _c(depth, np.float64)
    H, W = d.shape
    out = np.empty((2, H, W), np.float64)
    assert lib().orc_sobel_f64(_p(d), W, H, _p(out)) == 0
    return out


def philox4x32_10(ctr, key) -> np.ndarray:
    c = _c(ctr, np.uint32)
    k = _c(key, np.uint32)
    out = np.empty(4, np.uint32)
    lib().orc_philox4x32_10(_p(c), _p(k), _p(out))
    return out


def sample_triple(r0: int, r1: int, r2: int, n: int) -> tuple:
    out = np.empty(3, np.uint32)
    lib().orc_sample_triple(r0, r1, r2, n, _p(out))
    return tuple(int(x) for x in out)


def colex_unrank3(h: int, n: int):
    out = np.empty(3, np.uint32)
    ok = lib().orc_colex_unrank3(h, n, _p(out))
    return tuple(int(x) for x in out) if ok else None


def deproject(u: int, v: int, z: float, K) -> np.ndarray:
    out = np.empty(3, np.float32)
    lib().orc_deproject(u, v, z, K.fx, K.fy, K.cx, K.cy, _p(out))
    return out


def plane_from_3pts(p0, p1, p2):
    a, b, c = (_c(p, np.float32) for p in (p0, p1, p2))
    out = np.zeros(4, np.float32)
    ok = lib().orc_plane_from_3pts(_p(a), _p(b), _p(c), _p(out))
    return (out if ok else None)


def point_plane_dist(plane, P) -> float:
    pl = _c(plane, np.float32)
    q = _c(P, np.float32)
    return float(lib().orc_point_plane_dist(_p(pl), _p(q)))


def refit_plane(pts: np.ndarray):
    q = _c(pts, np.float64).reshape(-1, 3)
    out = np.zeros(7, np.float64)
    ok = lib().orc_refit_plane(_p(q), q.shape[0], _p(out))
    return out if ok else None


def ransac(depth: np.ndarray, labels: np.ndarray, K, n_regions: int, n_hyp: int, tau: float,
           seed: int, frame_id: int = 0, sampler: int = SAMPLER_PHILOX,
           select: int = SELECT_COUNT, debug: bool = False) -> dict:
    """Alg. 2 over every region of one frame.  Returns numpy arrays:
    n [R,3], d [R], centroid [R,3] (float64), inliers, n_points, best_hyp,
    status [R] (int32), errq [R] (uint64) and, with debug=True, the
    per-hypothesis counts [R, H] (int32, -1 = invalid) and errq_all [R, H]."""
    d = _c(depth, np.float32)
    lab = _c(labels, np.int32)
    H, W = d.shape
    assert lab.shape == (H, W)
    R = int(n_regions)
    of = np.zeros((max(R, 1), 7), np.float64)
    oi = np.zeros((max(R, 1), 4), np.int32)
    oe = np.zeros(max(R, 1), np.uint64)
    cnt = np.zeros((max(R, 1), n_hyp), np.int32) if debug else None
    ea = np.zeros((max(R, 1), n_hyp), np.uint64) if debug else None
    rc = lib().orc_ransac(_p(d), _p(lab), W, H, K.fx, K.fy, K.cx, K.cy, R, int(n_hyp), float(tau),
                          int(seed) & (2**64 - 1), int(frame_id), int(sampler), int(select),
                          _p(of), _p(oi), _p(oe),
                          _p(cnt) if debug else None, _p(ea) if debug else None)
    assert rc == 0
    res = dict(n=of[:R, 0:3], d=of[:R, 3], centroid=of[:R, 4:7], inliers=oi[:R, 0],
               n_points=oi[:R, 1], best_hyp=oi[:R, 2], status=oi[:R, 3], errq=oe[:R])
    if debug:
        res["counts"] = cnt[:R]
        res["errq_all"] = ea[:R]
    return res


def normals_to_u8(normals: np.ndarray) -> np.ndarray:
    """f32 [3, H, W] normals -> u8 [H, W, 3], c = rint((n + 1) * 127.5)."""
    n = _c(normals, np.float32)
    _, H, W = n.shape
    out = np.empty((H, W, 3), np.uint8)
    lib().orc_normals_to_u8(_p(n), W, H, _p(out))
    return out


def canny_u8(img: np.ndarray, low: float, high: float) -> np.ndarray:
    """Canny (L2, 3x3 Sobel, replicated border) on u8 [H, W] or [H, W, C] -> u8 0/255."""
    a = _c(img, np.uint8)
    H, W = a.shape[:2]
    C = 1 if a.ndim == 2 else a.shape[2]
    out = np.empty((H, W), np.uint8)
    assert lib().orc_canny_u8(_p(a), W, H, C, float(low), float(high), _p(out)) == 0
    return out


def segment_regions(normals: np.ndarray, low: float = 30.0, high: float = 90.0, min_area: int = 300,
                    max_regions: int = 1024):
    """NEXT-2 region labels from f32 normals [3, H, W]: (labels int32 [H, W],
    n_regions, dilated edge mask u8 [H, W])."""
    n = _c(normals, np.float32)
    _, H, W = n.shape
    labels = np.empty((H, W), np.int32)
    nr = np.zeros(1, np.int32)
    edges = np.empty((H, W), np.uint8)
    assert lib().orc_segment_regions(_p(n), W, H, float(low), float(high), int(min_area), int(max_regions),
                                     _p(labels), _p(nr), _p(edges)) == 0
    return labels, int(nr[0]), edges


# ---------------------------------------------------------------- NEXT-3
def trace_contour(labels: np.ndarray, region: int) -> np.ndarray:
    """Q35: outer boundary of `region` by Moore-neighbour tracing: int32 [n, 2] (x, y)."""
    lab = _c(labels, np.int32)
    H, W = lab.shape
    cap = 2 * (W + H) + 4 * int((lab == region).sum()) + 8
    pts = np.empty((cap, 2), np.int32)
    n = lib().orc_trace_contour(_p(lab), W, H, int(region), _p(pts), cap)
    assert n <= cap
    return pts[:n].copy()


def simplify_dp(pts: np.ndarray, eps: float, return_index: bool = False):
    """Q36: Douglas-Peucker on a closed integer contour [n, 2], eps in px
    (exact, eps rounded to 1/16 px): the kept points in contour order (and
    their contour indices)."""
    a = _c(pts, np.int32)
    keep = np.zeros(len(a), np.uint8)
    m = lib().orc_simplify_dp(_p(a), len(a), int(round(eps * 16)), _p(keep))
    idx = np.nonzero(keep)[0]
    assert len(idx) == m
    return (a[idx], idx) if return_index else a[idx]


def rasterize_polygons(polys, W: int, H: int) -> np.ndarray:
    """Q37/Q38: list of int32 [m, 2] vertex arrays -> label image int32 [H, W]."""
    offs, nv, vs = [], [], []
    o = 0
    for q in polys:
        q = np.asarray(q, np.int32).reshape(-1, 2)
        offs.append(o); nv.append(len(q)); vs.append(q)
        o += len(q)
    verts = np.ascontiguousarray(np.concatenate(vs) if vs else np.zeros((0, 2), np.int32), np.int32)
    offs = np.asarray(offs, np.int32); nv = np.asarray(nv, np.int32)
    out = np.empty((H, W), np.int32)
    assert lib().orc_rasterize_polygons(_p(verts), _p(offs), _p(nv), len(polys), W, H, _p(out)) == 0
    return out


def lift_vertices(uv: np.ndarray, plane, K) -> np.ndarray:
    """Q39: pixel vertices [n, 2] onto plane (nx, ny, nz, d) along camera rays -> [n, 3] f64."""
    a = _c(uv, np.int32)
    pl = np.asarray(plane, np.float64)
    X = np.empty((len(a), 3), np.float64)
    lib().orc_lift_vertices(_p(a), len(a), _p(pl), float(K.fx), float(K.fy), float(K.cx), float(K.cy), _p(X))
    return X
