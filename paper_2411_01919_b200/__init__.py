"""B200-native hot path of arXiv 2411.01919 (planar semantic mapping):
anisotropic diffusion + fused normals (Alg. 1) and batched RANSAC plane
fitting (Alg. 2), as hand-written sm_100a CUDA kernels behind the C ABI of
``include/pmap.h`` (``libpmap.so``).

This module is argument marshalling only: it passes device pointers of torch
tensors and the current CUDA stream to the C ABI; every step of the path runs
in the library's kernels.  There is no CPU fallback: importing this package
without the built library raises.
"""
from __future__ import annotations

import ctypes
import os
from typing import NamedTuple

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
# PMAP_LIB_VARIANT=<name> loads libpmap_<name>.so from the same directory
# (A/B kernel timing in tools/ only; default: the in-tree libpmap.so)
_VARIANT = os.environ.get("PMAP_LIB_VARIANT", "")
LIB_PATH = os.path.join(_HERE, f"libpmap_{_VARIANT}.so" if _VARIANT else "libpmap.so")

if not os.path.exists(LIB_PATH):
    raise ImportError(f"{LIB_PATH} is missing: build it with `make` (or __graft_entry__.build()); "
                      "this package has no CPU fallback")

_lib = ctypes.CDLL(LIB_PATH)

STATUS_OK, STATUS_REJECTED, STATUS_TOO_FEW, STATUS_DEGENERATE = 0, 1, 2, 3
SAMPLER_PHILOX, SAMPLER_ENUMERATE = 0, 1
SELECT_COUNT, SELECT_ERROR, SELECT_COUNT_EARLY, SELECT_ERROR_EARLY = 0, 1, 2, 3
ADF_ALG1, ADF_DIVERGENCE = 0, 1
NORMALS_GEOMETRIC, NORMALS_AS_PRINTED = 0, 1
ENGINE_AUTO, ENGINE_TILED, ENGINE_REG, ENGINE_HOLES = 0, 1, 3, 4
DEPTH_F32_M, DEPTH_U16_MM = 0, 1
LABELS_I32, LABELS_U16, LABELS_U8, LABELS_RUNS = 0, 1, 2, 3
PLANE_WORDS = 12          # sizeof(pm_plane) / 4


class pm_intrinsics(ctypes.Structure):
    _fields_ = [("fx", ctypes.c_float), ("fy", ctypes.c_float), ("cx", ctypes.c_float), ("cy", ctypes.c_float)]


class pm_adf_options(ctypes.Structure):
    _fields_ = [("iters_per_pass", ctypes.c_int32), ("scheme", ctypes.c_int32), ("normals_mode", ctypes.c_int32),
                ("engine", ctypes.c_int32)]


class pm_segment_params(ctypes.Structure):
    _fields_ = [("canny_low", ctypes.c_float), ("canny_high", ctypes.c_float), ("min_area", ctypes.c_int32),
                ("max_regions", ctypes.c_int32)]


class pm_ransac_options(ctypes.Structure):
    _fields_ = [("sampler", ctypes.c_int32), ("select", ctypes.c_int32),
                ("counts_out", ctypes.c_void_p), ("errq_out", ctypes.c_void_p),
                ("stage_events", ctypes.c_void_p)]


RANSAC_STAGE_EVENTS = 6


_P, _I32, _U32, _U64, _F32, _SZ = (ctypes.c_void_p, ctypes.c_int32, ctypes.c_uint32, ctypes.c_uint64,
                                   ctypes.c_float, ctypes.c_size_t)
_KP = ctypes.POINTER(pm_intrinsics)
_lib.pm_status_string.restype = ctypes.c_char_p
_lib.pm_status_string.argtypes = [ctypes.c_int]
_lib.pm_version.restype = _I32
_lib.pm_pipeline_kernel_launches.restype = _I32
_lib.pm_pipeline_kernel_launches.argtypes = [_I32, _I32]
_lib.pm_adf_workspace_bytes.restype = _SZ
_lib.pm_adf_workspace_bytes.argtypes = [_I32, _I32, _I32]
_lib.pm_ransac_workspace_bytes.restype = _SZ
_lib.pm_ransac_workspace_bytes.argtypes = [_I32, _I32, _I32, _I32, _I32]
_lib.pm_pipeline_workspace_bytes.restype = _SZ
_lib.pm_pipeline_workspace_bytes.argtypes = [_I32, _I32, _I32, _I32, _I32]
_lib.pm_adf_filter.argtypes = [_P, _P, _I32, _I32, _KP, _F32, _F32, _I32, _P, _P, _SZ, _P]
_lib.pm_adf_filter_batched.argtypes = [_P, _P, _I32, _I32, _I32, _KP, _F32, _F32, _I32, _P, _P, _SZ, _P]
_lib.pm_adf_filter_ex.argtypes = [_P, _P, _I32, _I32, _I32, _KP, _F32, _F32, _I32, _P, _P, _SZ,
                                  ctypes.POINTER(pm_adf_options), _P]
_lib.pm_normals_from_depth.argtypes = [_P, _I32, _I32, _KP, _P, _P]
_lib.pm_normals_from_depth_batched.argtypes = [_P, _I32, _I32, _I32, _KP, _P, _P]
_lib.pm_normals_from_depth_ex.argtypes = [_P, _I32, _I32, _I32, _KP, _I32, _P, _P]
_lib.pm_ransac_planes.argtypes = [_P, _I32, _I32, _KP, _P, _I32, _I32, _F32, _U64, _P, _P, _SZ, _P]
_lib.pm_ransac_planes_batched.argtypes = [_P, _I32, _I32, _I32, _U32, _KP, _P, _I32, _I32, _F32, _U64,
                                          _P, _P, _SZ, _P]
_lib.pm_ransac_planes_ex.argtypes = [_P, _I32, _I32, _I32, _U32, _KP, _P, _I32, _I32, _F32, _U64, _P, _P, _SZ,
                                     ctypes.POINTER(pm_ransac_options), _P]
_lib.pm_process_frames.argtypes = [_P, _P, _I32, _I32, _I32, _U32, _KP, _F32, _F32, _I32, _I32, _I32, _F32,
                                   _U64, _P, _P, _P, _P, _SZ, _P]
_lib.pm_process_frames_host_async.argtypes = [_P, _I32, _P, _I32, _I32, _I32, _I32, _U32, _KP, _F32, _F32, _I32,
                                              _I32, _I32, _F32, _U64, _P, _P, _P, _I32, _P, _SZ, _P]
_lib.pm_process_frames_host_async.restype = ctypes.c_int
_lib.pm_process_frames_host.argtypes = [_P, _I32, _P, _I32, _I32, _I32, _I32, _U32, _KP, _F32, _F32, _I32, _I32,
                                        _I32, _F32, _U64, _P, _P, _P, _I32, _P, _SZ, _P]
_lib.pm_host_pipeline_arena_bytes.restype = _SZ
_lib.pm_host_pipeline_arena_bytes.argtypes = [_I32, _I32, _I32, _I32, _I32, _I32, _I32]
_lib.pm_depth_u16_to_metres.argtypes = [_P, _P, _SZ, _F32, _P]
_lib.pm_segment_regions.argtypes = [_P, _I32, _I32, _I32, ctypes.POINTER(pm_segment_params), _P, _P, _P, _P, _SZ, _P]
_lib.pm_segment_workspace_bytes.restype = _SZ
_lib.pm_segment_workspace_bytes.argtypes = [_I32, _I32, _I32, _I32]
for _fn in ("pm_adf_filter", "pm_adf_filter_batched", "pm_adf_filter_ex", "pm_normals_from_depth",
            "pm_normals_from_depth_batched", "pm_normals_from_depth_ex", "pm_ransac_planes",
            "pm_ransac_planes_batched", "pm_ransac_planes_ex", "pm_process_frames", "pm_process_frames_host",
            "pm_depth_u16_to_metres", "pm_segment_regions"):
    getattr(_lib, _fn).restype = ctypes.c_int

EXPORTED = ("pm_adf_filter", "pm_adf_filter_batched", "pm_adf_filter_ex", "pm_adf_workspace_bytes",
            "pm_normals_from_depth", "pm_normals_from_depth_batched", "pm_normals_from_depth_ex", "pm_ransac_planes",
            "pm_ransac_planes_batched", "pm_ransac_planes_ex", "pm_ransac_workspace_bytes",
            "pm_process_frames", "pm_pipeline_workspace_bytes", "pm_pipeline_kernel_launches",
            "pm_process_frames_host", "pm_process_frames_host_async", "pm_host_pipeline_arena_bytes",
            "pm_depth_u16_to_metres",
            "pm_segment_regions", "pm_segment_workspace_bytes",
            "pm_region_polygons", "pm_region_polygons_workspace_bytes", "pm_rasterize_polygons",
            "pm_lift_polygon_vertices",
            "pm_drift_kalman_step", "pm_merge_gate", "pm_plane_map_merge_frame",
            "pm_status_string", "pm_version")


class PMError(RuntimeError):
    pass


def _check(rc: int) -> None:
    if rc != 0:
        raise PMError(f"pmap: {_lib.pm_status_string(rc).decode()} (status {rc})")


def version() -> int:
    return int(_lib.pm_version())


def _K(K) -> pm_intrinsics:
    if isinstance(K, pm_intrinsics):
        return K
    if isinstance(K, (tuple, list)):
        return pm_intrinsics(*[float(x) for x in K])
    return pm_intrinsics(float(K.fx), float(K.fy), float(K.cx), float(K.cy))


def _frames(t: torch.Tensor, dtype) -> tuple:
    if not t.is_cuda:
        raise PMError("pmap: tensors must live on a CUDA device")
    if t.dtype != dtype or not t.is_contiguous():
        raise PMError(f"pmap: expected a contiguous {dtype} tensor")
    if t.dim() == 2:
        return 1, t.shape[0], t.shape[1]
    if t.dim() == 3:
        return t.shape[0], t.shape[1], t.shape[2]
    raise PMError("pmap: expected [H, W] or [B, H, W]")


def _stream(t: torch.Tensor) -> int:
    return torch.cuda.current_stream(t.device).cuda_stream


def _workspace(nbytes: int, device) -> torch.Tensor:
    return torch.empty(max(int(nbytes), 256), dtype=torch.uint8, device=device)


def _out(t, shape, dtype, device, name: str) -> torch.Tensor:
    """Allocate an output, or check a caller's: same device, dtype, contiguous,
    exactly the element count the call writes (the library trusts pointers)."""
    if t is None:
        return torch.empty(shape, dtype=dtype, device=device)
    n = 1
    for d in shape:
        n *= int(d)
    if t.device != device or t.dtype != dtype or not t.is_contiguous() or t.numel() != n:
        raise PMError(f"pmap: {name} must be a contiguous {dtype} tensor of {n} elements on {device}")
    return t


def _ws(t, nbytes: int, device, name: str = "workspace") -> torch.Tensor:
    """A caller's workspace must be contiguous uint8 memory on the call's
    device (the library checks its size and alignment)."""
    if t is None:
        return _workspace(nbytes, device)
    if t.device != device or t.dtype != torch.uint8 or not t.is_contiguous():
        raise PMError(f"pmap: {name} must be a contiguous uint8 tensor on {device}")
    return t


def _same_shape(a: torch.Tensor, b: torch.Tensor, what: str) -> None:
    if tuple(a.shape) != tuple(b.shape) or a.device != b.device:
        raise PMError(f"pmap: {what} must have the depth's shape and device")


def pipeline_kernel_launches(iters: int, n_regions: int) -> int:
    return int(_lib.pm_pipeline_kernel_launches(int(iters), int(n_regions)))


def adf_workspace_bytes(W: int, H: int, n_frames: int = 1) -> int:
    return int(_lib.pm_adf_workspace_bytes(W, H, n_frames))


def ransac_workspace_bytes(W: int, H: int, n_regions: int, n_hyp: int, n_frames: int = 1) -> int:
    return int(_lib.pm_ransac_workspace_bytes(W, H, n_regions, n_hyp, n_frames))


def pipeline_workspace_bytes(W: int, H: int, n_regions: int, n_hyp: int, n_frames: int = 1) -> int:
    return int(_lib.pm_pipeline_workspace_bytes(W, H, n_regions, n_hyp, n_frames))


def adf_filter(depth: torch.Tensor, K, lam: float, kappa: float, iters: int, normals: bool = True,
               iters_per_pass: int = 0, out: torch.Tensor = None, normals_out: torch.Tensor = None,
               workspace: torch.Tensor = None, scheme: int = ADF_ALG1, normals_mode: int = NORMALS_GEOMETRIC,
               engine: int = ENGINE_AUTO):
    """Alg. 1 on [H, W] or [B, H, W] f32 depth (metres, CUDA).
    Returns (I_smooth, normals [.., 3, H, W] or None)."""
    B, H, W = _frames(depth, torch.float32)
    dev = depth.device
    out = _out(out, depth.shape, torch.float32, dev, "out")
    nrm = None
    if normals:
        shape = (3, H, W) if depth.dim() == 2 else (B, 3, H, W)
        nrm = _out(normals_out, shape, torch.float32, dev, "normals_out")
    ws = _ws(workspace, adf_workspace_bytes(W, H, B), dev)
    opt = pm_adf_options(int(iters_per_pass), int(scheme), int(normals_mode), int(engine))
    with torch.cuda.device(dev):
        _check(_lib.pm_adf_filter_ex(depth.data_ptr(), out.data_ptr(), W, H, B, ctypes.byref(_K(K)), float(lam),
                                     float(kappa), int(iters), nrm.data_ptr() if nrm is not None else None,
                                     ws.data_ptr(), ws.numel(), ctypes.byref(opt), _stream(depth)))
    return out, nrm


def normals_from_depth(depth: torch.Tensor, K, out: torch.Tensor = None, mode: int = NORMALS_GEOMETRIC) -> torch.Tensor:
    """Alg. 1 ℓ9-13 on [H, W] or [B, H, W] f32 depth -> [.., 3, H, W]."""
    B, H, W = _frames(depth, torch.float32)
    shape = (3, H, W) if depth.dim() == 2 else (B, 3, H, W)
    out = _out(out, shape, torch.float32, depth.device, "out")
    with torch.cuda.device(depth.device):
        _check(_lib.pm_normals_from_depth_ex(depth.data_ptr(), W, H, B, ctypes.byref(_K(K)), int(mode),
                                             out.data_ptr(), _stream(depth)))
    return out


class Planes(NamedTuple):
    """Views of a pm_plane table [.., R] (48-byte records)."""
    raw: torch.Tensor        # int32 [.., R, 12]

    @property
    def n(self):
        return self.raw[..., 0:3].view(torch.float32)

    @property
    def d(self):
        return self.raw[..., 3].view(torch.float32)

    @property
    def centroid(self):
        return self.raw[..., 4:7].view(torch.float32)

    @property
    def inliers(self):
        return self.raw[..., 7]

    @property
    def n_points(self):
        return self.raw[..., 8]

    @property
    def best_hyp(self):
        return self.raw[..., 9]

    @property
    def status(self):
        return self.raw[..., 10]

    @property
    def sum_dist(self):
        return self.raw[..., 11].view(torch.float32)


def ransac_planes(depth: torch.Tensor, K, labels: torch.Tensor, n_regions: int, n_hyp: int, tau: float,
                  seed: int, first_frame_id: int = 0, sampler: int = SAMPLER_PHILOX,
                  select: int = SELECT_COUNT, debug: bool = False, out: torch.Tensor = None,
                  workspace: torch.Tensor = None, stage_events=None):
    """Alg. 2 over every region of every frame.  Returns Planes
    (and, with debug=True, per-hypothesis counts / errq tensors [.., R, n_hyp];
    debug="counts": counts only, errq None -- the scoring kernel without the
    error sums, i.e. the one the default call runs)."""
    B, H, W = _frames(depth, torch.float32)
    _same_shape(labels, depth, "labels")
    _frames(labels, torch.int32)
    lead = () if depth.dim() == 2 else (B,)
    out = _out(out, lead + (n_regions, PLANE_WORDS), torch.int32, depth.device, "out")
    ws = _ws(workspace, ransac_workspace_bytes(W, H, n_regions, n_hyp, B), depth.device)
    counts = errq = None
    if debug:
        counts = torch.empty(lead + (n_regions, n_hyp), dtype=torch.int32, device=depth.device)
    if debug and debug != "counts":   # "counts": counts only (keeps the default scoring kernel)
        errq = torch.empty(lead + (n_regions, n_hyp), dtype=torch.int64, device=depth.device)
    ev_arr = None
    if stage_events is not None:   # RANSAC_STAGE_EVENTS torch.cuda.Event objects (timing)
        if len(stage_events) != RANSAC_STAGE_EVENTS:
            raise PMError(f"pmap: stage_events needs {RANSAC_STAGE_EVENTS} events")
        ev_arr = (ctypes.c_void_p * RANSAC_STAGE_EVENTS)(*[e.cuda_event for e in stage_events])
    opt = pm_ransac_options(int(sampler), int(select), counts.data_ptr() if counts is not None else None,
                            errq.data_ptr() if errq is not None else None,
                            ctypes.cast(ev_arr, ctypes.c_void_p) if ev_arr is not None else None)
    with torch.cuda.device(depth.device):
        _check(_lib.pm_ransac_planes_ex(depth.data_ptr(), W, H, B, int(first_frame_id), ctypes.byref(_K(K)),
                                        labels.data_ptr(), int(n_regions), int(n_hyp), float(tau),
                                        int(seed) & (2**64 - 1), out.data_ptr(), ws.data_ptr(), ws.numel(),
                                        ctypes.byref(opt), _stream(depth)))
    planes = Planes(out)
    return (planes, counts, errq) if debug else planes


def process_frames(depth: torch.Tensor, labels: torch.Tensor, K, lam: float, kappa: float, iters: int,
                   n_regions: int, n_hyp: int, tau: float, seed: int, first_frame_id: int = 0,
                   depth_out: torch.Tensor = None, normals_out: torch.Tensor = None,
                   planes_out: torch.Tensor = None, workspace: torch.Tensor = None):
    """The whole per-frame path in one C-ABI call (pm_process_frames):
    adf_filter with fused normals, then ransac_planes on the filtered depth."""
    B, H, W = _frames(depth, torch.float32)
    _same_shape(labels, depth, "labels")
    _frames(labels, torch.int32)
    lead = () if depth.dim() == 2 else (B,)
    dev = depth.device
    depth_out = _out(depth_out, depth.shape, torch.float32, dev, "depth_out")
    normals_out = _out(normals_out, lead + (3, H, W), torch.float32, dev, "normals_out")
    planes_out = _out(planes_out, lead + (n_regions, PLANE_WORDS), torch.int32, dev, "planes_out")
    ws = _ws(workspace, pipeline_workspace_bytes(W, H, n_regions, n_hyp, B), dev)
    with torch.cuda.device(dev):
        _check(_lib.pm_process_frames(depth.data_ptr(), labels.data_ptr(), W, H, B, int(first_frame_id),
                                      ctypes.byref(_K(K)), float(lam), float(kappa), int(iters), int(n_regions),
                                      int(n_hyp), float(tau), int(seed) & (2**64 - 1), depth_out.data_ptr(),
                                      normals_out.data_ptr(), planes_out.data_ptr(), ws.data_ptr(), ws.numel(),
                                      _stream(depth)))
    return depth_out, normals_out, Planes(planes_out)


def host_pipeline_arena_bytes(W: int, H: int, n_regions: int, n_hyp: int, chunk_frames: int,
                              depth_format: int = DEPTH_F32_M, label_format: int = LABELS_I32) -> int:
    return int(_lib.pm_host_pipeline_arena_bytes(W, H, n_regions, n_hyp, chunk_frames, depth_format, label_format))


def depth_u16_to_metres(depth_mm: torch.Tensor, out: torch.Tensor = None, scale: float = 1e-3) -> torch.Tensor:
    """uint16 millimetres -> f32 metres on the device (0 stays 0 = invalid)."""
    if depth_mm.dtype != torch.uint16 or not depth_mm.is_cuda or not depth_mm.is_contiguous():
        raise PMError("pmap: expected a contiguous CUDA uint16 tensor")
    out = _out(out, depth_mm.shape, torch.float32, depth_mm.device, "out")
    with torch.cuda.device(depth_mm.device):
        _check(_lib.pm_depth_u16_to_metres(depth_mm.data_ptr(), out.data_ptr(), depth_mm.numel(), float(scale),
                                           _stream(out)))
    return out


class pm_label_runs(ctypes.Structure):
    _fields_ = [("row_start", ctypes.c_void_p), ("runs", ctypes.c_void_p)]


class LabelRuns(NamedTuple):
    """Row run-length region labels of [B, H, W] frames (host tensors, int32
    storage of the uint32 words of include/pmap.h pm_label_runs)."""
    row_start: torch.Tensor   # [B*H + 1]
    runs: torch.Tensor        # [n_runs]: label (low 16 bits, 0xFFFF = none) | length << 16
    shape: tuple              # (B, H, W)

    def pin_memory(self):
        return LabelRuns(self.row_start.pin_memory(), self.runs.pin_memory(), self.shape)

    @property
    def nbytes(self) -> int:
        return 4 * (self.row_start.numel() + self.runs.numel())


def encode_label_runs(labels: torch.Tensor) -> LabelRuns:
    """[B, H, W] integer labels (negative or >= 0xFFFF = none) -> LabelRuns
    (host side, vectorised): one run per maximal constant stretch of a row."""
    import numpy as np
    a = labels.detach().cpu().numpy().astype(np.int64)
    if a.ndim != 3:
        raise PMError("pmap: expected [B, H, W] labels")
    B, H, W = a.shape
    if W > 65535:
        raise PMError("pmap: run lengths are 16-bit (W <= 65535)")
    lab = np.where((a < 0) | (a >= 0xFFFF), 0xFFFF, a).reshape(B * H, W)
    start = np.ones((B * H, W), bool)
    start[:, 1:] = lab[:, 1:] != lab[:, :-1]
    r_idx, c_idx = np.nonzero(start)                     # run starts, raster order
    row_start = np.zeros(B * H + 1, np.uint32)
    row_start[1:] = np.cumsum(start.sum(1), dtype=np.uint64).astype(np.uint32)
    end = np.empty_like(c_idx)
    end[:-1] = c_idx[1:]
    end[-1] = W
    last = np.ones(len(c_idx), bool)
    last[:-1] = r_idx[1:] != r_idx[:-1]
    end[last] = W
    runs = lab[r_idx, c_idx].astype(np.uint32) | ((end - c_idx).astype(np.uint32) << 16)
    return LabelRuns(torch.from_numpy(row_start.view(np.int32).copy()), torch.from_numpy(runs.view(np.int32).copy()),
                     (B, H, W))


def process_frames_host(depth: torch.Tensor, labels, K, lam: float, kappa: float, iters: int,
                        n_regions: int, n_hyp: int, tau: float, seed: int, first_frame_id: int = 0,
                        chunk_frames: int = 64, planes_out: torch.Tensor = None, depth_out: torch.Tensor = None,
                        normals_out: torch.Tensor = None, arena: torch.Tensor = None, device=None,
                        sync: bool = True):
    """pm_process_frames_host: CPU (preferably pinned) tensors in, CPU plane
    table out.  depth: [B, H, W] float32 metres or uint16 millimetres; labels:
    [B, H, W] int32, uint16 (0xFFFF = none) or uint8 (0xFF = none), or a
    LabelRuns (encode_label_runs).  sync=False: pm_process_frames_host_async
    -- returns once queued; the host tensors, planes_out and the arena (both
    required then) must stay untouched until the device's current stream is
    synchronised; consecutive calls overlap."""
    runs = labels if isinstance(labels, LabelRuns) else None
    if depth.is_cuda or (runs is None and labels.is_cuda):
        raise PMError("pmap: process_frames_host takes host tensors")
    if depth.dim() != 3 or tuple(runs.shape if runs is not None else labels.shape) != tuple(depth.shape):
        raise PMError("pmap: expected [B, H, W] depth and labels")
    dfmt = {torch.float32: DEPTH_F32_M, torch.uint16: DEPTH_U16_MM}.get(depth.dtype)
    if runs is not None:
        lfmt = LABELS_RUNS
        if runs.row_start.is_cuda or runs.runs.is_cuda or runs.row_start.dtype != torch.int32 or \
                runs.runs.dtype != torch.int32 or not runs.row_start.is_contiguous() or \
                not runs.runs.is_contiguous() or runs.row_start.numel() != depth.shape[0] * depth.shape[1] + 1:
            raise PMError("pmap: LabelRuns must hold contiguous host int32 row_start [B*H+1] and runs")
        lab_arg = pm_label_runs(runs.row_start.data_ptr(), runs.runs.data_ptr())
    else:
        lfmt = {torch.int32: LABELS_I32, torch.uint16: LABELS_U16, torch.uint8: LABELS_U8}.get(labels.dtype)
        if lfmt is not None and not labels.is_contiguous():
            lfmt = None
    if dfmt is None or lfmt is None or not depth.is_contiguous():
        raise PMError("pmap: depth float32|uint16, labels int32|uint16|uint8|LabelRuns, contiguous")
    B, H, W = depth.shape
    dev = torch.device("cuda") if device is None else torch.device(device)
    C = min(int(chunk_frames), B)
    if dev.type == "cuda" and dev.index is None:
        dev = torch.device("cuda", torch.cuda.current_device())
    if not sync and (arena is None or planes_out is None):
        raise PMError("pmap: sync=False needs a caller-owned arena and planes_out (they outlive the call)")
    arena = _ws(arena, 0, dev, "arena") if arena is not None else torch.empty(
        host_pipeline_arena_bytes(W, H, n_regions, n_hyp, C, dfmt, lfmt), dtype=torch.uint8, device=dev)
    cpu = torch.device("cpu")
    planes_out = _out(planes_out, (B, n_regions, PLANE_WORDS), torch.int32, cpu, "planes_out")
    if depth_out is not None:
        depth_out = _out(depth_out, (B, H, W), torch.float32, cpu, "depth_out")
    if normals_out is not None:
        normals_out = _out(normals_out, (B, 3, H, W), torch.float32, cpu, "normals_out")
    with torch.cuda.device(dev):
        stream = torch.cuda.current_stream(dev).cuda_stream
        lab_ptr = ctypes.addressof(lab_arg) if runs is not None else labels.data_ptr()
        fn = _lib.pm_process_frames_host if sync else _lib.pm_process_frames_host_async
        _check(fn(depth.data_ptr(), dfmt, lab_ptr, lfmt, W, H, B,
                                           int(first_frame_id), ctypes.byref(_K(K)), float(lam), float(kappa),
                                           int(iters), int(n_regions), int(n_hyp), float(tau),
                                           int(seed) & (2**64 - 1), planes_out.data_ptr(),
                                           depth_out.data_ptr() if depth_out is not None else None,
                                           normals_out.data_ptr() if normals_out is not None else None, C,
                                           arena.data_ptr(), arena.numel(), stream))
    return Planes(planes_out)


def segment_workspace_bytes(W: int, H: int, n_frames: int = 1, min_area: int = 300) -> int:
    return int(_lib.pm_segment_workspace_bytes(W, H, n_frames, min_area))


def segment_regions(normals: torch.Tensor, canny_low: float = 30.0, canny_high: float = 90.0, min_area: int = 300,
                    max_regions: int = 1024, edges: bool = False, workspace: torch.Tensor = None):
    """NEXT-2: region labels from a [3, H, W] / [B, 3, H, W] f32
    normal image.  Returns (labels int32 [.., H, W], n_regions int32 [B],
    edge mask uint8 [.., H, W] or None)."""
    if not normals.is_cuda or normals.dtype != torch.float32 or not normals.is_contiguous():
        raise PMError("pmap: expected a contiguous CUDA float32 normal image")
    single = normals.dim() == 3
    n4 = normals.unsqueeze(0) if single else normals
    B, C, H, W = n4.shape
    if C != 3:
        raise PMError("pmap: expected 3 normal channels")
    dev = normals.device
    labels = torch.empty(B, H, W, dtype=torch.int32, device=dev)
    nreg = torch.empty(B, dtype=torch.int32, device=dev)
    emask = torch.empty(B, H, W, dtype=torch.uint8, device=dev) if edges else None
    ws = _ws(workspace, segment_workspace_bytes(W, H, B, min_area), dev)
    prm = pm_segment_params(float(canny_low), float(canny_high), int(min_area), int(max_regions))
    with torch.cuda.device(dev):
        _check(_lib.pm_segment_regions(n4.data_ptr(), W, H, B, ctypes.byref(prm), labels.data_ptr(),
                                       nreg.data_ptr(), emask.data_ptr() if edges else None, ws.data_ptr(),
                                       ws.numel(), _stream(normals)))
    if single:
        labels = labels[0]
        emask = emask[0] if edges else None
    return labels, nreg, emask


# ---------------------------------------------------------------- NEXT-4 (host)
class pm_drift_filter(ctypes.Structure):
    _fields_ = [("x", ctypes.c_double), ("P", ctypes.c_double)]


class pm_map_plane(ctypes.Structure):
    _fields_ = [("n", ctypes.c_double * 3), ("c", ctypes.c_double * 3), ("w", ctypes.c_double),
                ("n_obs", ctypes.c_int32), ("pad", ctypes.c_int32)]


class pm_map_params(ctypes.Structure):
    _fields_ = [("drift_tol", ctypes.c_double), ("normal_tol", ctypes.c_double), ("xy_radius", ctypes.c_double),
                ("sigma_p", ctypes.c_double), ("sigma_m", ctypes.c_double)]


_lib.pm_drift_kalman_step.restype = ctypes.c_double
_lib.pm_drift_kalman_step.argtypes = [ctypes.POINTER(pm_drift_filter), ctypes.c_double, ctypes.c_double,
                                      ctypes.c_double]
_lib.pm_merge_gate.restype = _I32
_lib.pm_merge_gate.argtypes = [ctypes.c_double, ctypes.c_double, ctypes.c_double, ctypes.POINTER(ctypes.c_double)]
_lib.pm_plane_map_merge_frame.restype = ctypes.c_int


def drift_kalman_step(f: pm_drift_filter, z: float, sigma_p: float, sigma_m: float) -> float:
    """Eqs. 6-10 on the host; updates f, returns the gain K."""
    return float(_lib.pm_drift_kalman_step(ctypes.byref(f), float(z), float(sigma_p), float(sigma_m)))


def merge_gate(z_new: float, z_map: float, drift_tol: float = 0.05):
    """Eqs. 4-5: (dz, merge?)."""
    dz = ctypes.c_double()
    ok = _lib.pm_merge_gate(float(z_new), float(z_map), float(drift_tol), ctypes.byref(dz))
    return dz.value, bool(ok)


class PlaneMap:
    """Host-side plane map with drift compensation (NEXT-4): wraps
    pm_plane_map_merge_frame over a fixed-capacity pm_map_plane array."""

    def __init__(self, capacity: int = 4096, drift_tol: float = 0.05, normal_tol: float = 0.1745,
                 xy_radius: float = 0.5, sigma_p: float = 1e-4, sigma_m: float = 1e-4, P0: float = 1.0):
        self.capacity = int(capacity)
        self.planes = (pm_map_plane * self.capacity)()
        self.count = ctypes.c_int32(0)
        self.filter = pm_drift_filter(0.0, float(P0))
        self.params = pm_map_params(drift_tol, normal_tol, xy_radius, sigma_p, sigma_m)

    def merge_frame(self, plane_table: torch.Tensor, pose):
        """plane_table: int32 [R, 12] raw pm_plane rows (Planes.raw of one
        frame, any device); pose: 16 floats, row-major camera-to-world.
        Returns (match [R] list, z_k or None)."""
        raw = plane_table.detach().to("cpu", torch.int32).contiguous()
        R = raw.shape[0]
        pose_c = (ctypes.c_double * 16)(*[float(v) for v in pose])
        match = (ctypes.c_int32 * max(R, 1))()
        zk = ctypes.c_double()
        _check(_lib.pm_plane_map_merge_frame(self.planes, ctypes.byref(self.count), self.capacity,
                                             ctypes.c_void_p(raw.data_ptr()), R, pose_c, ctypes.byref(self.filter),
                                             ctypes.byref(self.params), match, ctypes.byref(zk)))
        z = zk.value
        return list(match)[:R], (None if z != z else z)

    def as_list(self):
        return [{"n": list(p.n), "c": list(p.c), "w": p.w, "n_obs": p.n_obs}
                for p in self.planes[:self.count.value]]


# ---------------------------------------------------------------- NEXT-3
class pm_polygon_params(ctypes.Structure):
    _fields_ = [("eps16", _I32), ("max_contour", _I32), ("max_vertices", _I32)]


_lib.pm_region_polygons.restype = ctypes.c_int
_lib.pm_rasterize_polygons.restype = ctypes.c_int
_lib.pm_lift_polygon_vertices.restype = ctypes.c_int
_lib.pm_region_polygons_workspace_bytes.restype = _SZ
_lib.pm_region_polygons_workspace_bytes.argtypes = [_I32, _I32, _I32]


class Polygons(NamedTuple):
    contour_len: torch.Tensor   # int32 [.., R]
    vertices: torch.Tensor      # int32 [.., R, max_vertices, 2]
    n_vertices: torch.Tensor    # int32 [.., R]


def region_polygons(labels: torch.Tensor, n_regions: int, eps: float = 3.0, max_contour: int = 8192,
                    max_vertices: int = 256, workspace: torch.Tensor = None) -> Polygons:
    """NEXT-3: outer contour of every region (Moore
    tracing) simplified by closed Douglas-Peucker (eps px, exact to 1/16 px)."""
    B, H, W = _frames(labels, torch.int32)
    lead = () if labels.dim() == 2 else (B,)
    dev = labels.device
    clen = torch.empty(lead + (n_regions,), dtype=torch.int32, device=dev)
    verts = torch.zeros(lead + (n_regions, max_vertices, 2), dtype=torch.int32, device=dev)
    nv = torch.empty(lead + (n_regions,), dtype=torch.int32, device=dev)
    nb = int(_lib.pm_region_polygons_workspace_bytes(B, n_regions, max_contour))
    ws = _ws(workspace, nb, dev)
    prm = pm_polygon_params(int(round(eps * 16)), int(max_contour), int(max_vertices))
    with torch.cuda.device(dev):
        _check(_lib.pm_region_polygons(ctypes.c_void_p(labels.data_ptr()), W, H, B, int(n_regions),
                                       ctypes.byref(prm), ctypes.c_void_p(clen.data_ptr()),
                                       ctypes.c_void_p(verts.data_ptr()), ctypes.c_void_p(nv.data_ptr()),
                                       ctypes.c_void_p(ws.data_ptr()), ctypes.c_size_t(ws.numel()),
                                       ctypes.c_void_p(_stream(labels))))
    return Polygons(clen, verts, nv)


def rasterize_polygons(polys: Polygons, W: int, H: int, out: torch.Tensor = None) -> torch.Tensor:
    """Labels [.., H, W] from polygons (lowest region index wins, -1 = none)."""
    v, nv = polys.vertices, polys.n_vertices
    single = nv.dim() == 1
    B = 1 if single else nv.shape[0]
    R, MV = v.shape[-3], v.shape[-2]
    out = _out(out, ((H, W) if single else (B, H, W)), torch.int32, v.device, "out")
    ws = _workspace(16 * B * max(R, 1), v.device)
    with torch.cuda.device(v.device):
        _check(_lib.pm_rasterize_polygons(ctypes.c_void_p(v.data_ptr()), ctypes.c_void_p(nv.data_ptr()), MV, W, H,
                                          B, R, ctypes.c_void_p(out.data_ptr()), ctypes.c_void_p(ws.data_ptr()),
                                          ctypes.c_size_t(ws.numel()), ctypes.c_void_p(_stream(v))))
    return out


def lift_polygon_vertices(polys: Polygons, planes, K) -> torch.Tensor:
    """Polygon vertices onto their region planes along camera rays: float64 [.., R, max_vertices, 3]."""
    v, nv = polys.vertices, polys.n_vertices
    single = nv.dim() == 1
    B = 1 if single else nv.shape[0]
    R, MV = v.shape[-3], v.shape[-2]
    raw = planes.raw if hasattr(planes, "raw") else planes
    if raw.device != v.device or raw.dtype != torch.int32 or not raw.is_contiguous() or \
            raw.numel() != B * R * PLANE_WORDS:
        raise PMError("pmap: planes must be the contiguous int32 plane table of the polygons' frames and regions")
    X = torch.empty(v.shape[:-1] + (3,), dtype=torch.float64, device=v.device)
    with torch.cuda.device(v.device):
        _check(_lib.pm_lift_polygon_vertices(ctypes.c_void_p(v.data_ptr()), ctypes.c_void_p(nv.data_ptr()), MV,
                                             ctypes.c_void_p(raw.data_ptr()), B, R, ctypes.byref(_K(K)),
                                             ctypes.c_void_p(X.data_ptr()), ctypes.c_void_p(_stream(v))))
    return X
