"""The C-ABI library loads and exports every symbol include/pmap.h declares;
host-side argument checks and workspace sizing (no compute calls, no GPU)."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "pmap.h")).read()
    return sorted(set(re.findall(r"PM_API\s+[\w\s\*]+?\b(pm_\w+)\s*\(", src)))


@pytest.fixture(scope="module")
def pm():
    import paper_2411_01919_b200 as pm
    return pm


def test_header_symbols_exported(pm):
    names = _declared()
    assert len(names) >= 14
    for n in names:
        assert hasattr(pm._lib, n), n
    assert set(names) == set(pm.EXPORTED)


def test_version_and_status_strings(pm):
    assert pm.version() >= 100
    assert pm._lib.pm_status_string(0) == b"ok"
    assert b"argument" in pm._lib.pm_status_string(1)


def test_workspace_sizing(pm):
    a = pm.adf_workspace_bytes(640, 480, 1)
    assert a >= 640 * 480 * 4 and a % 256 == 0
    assert pm.adf_workspace_bytes(640, 480, 8) >= 8 * 640 * 480 * 4
    r = pm.ransac_workspace_bytes(640, 480, 64, 64, 1)
    assert r >= 640 * 480 * 8 + 64 * 64 * (16 + 4 + 8)
    assert pm.ransac_workspace_bytes(640, 480, 64, 64, 4) >= 4 * 640 * 480 * 8
    assert pm.pipeline_workspace_bytes(640, 480, 64, 64, 1) == max(a, r)
    assert pm.ransac_workspace_bytes(0, 480, 64, 64, 1) == 0


def test_invalid_arguments_rejected_before_launch(pm):
    L = pm._lib
    K = pm.pm_intrinsics(385.0, 385.0, 319.5, 239.5)
    bogus = ctypes.c_void_p(0x1000)
    other = ctypes.c_void_p(0x100000000)
    INV = 1
    # null pointers / bad sizes / bad parameters (Alg. 1 requires gamma in (0, 1/4], k > 0)
    assert L.pm_adf_filter(None, other, 640, 480, ctypes.byref(K), 0.15, 0.03, 20, None, None, 0, None) == INV
    assert L.pm_adf_filter(bogus, other, 2, 480, ctypes.byref(K), 0.15, 0.03, 20, None, None, 0, None) == INV
    assert L.pm_adf_filter(bogus, other, 640, 480, ctypes.byref(K), 0.3, 0.03, 20, None, None, 0, None) == INV
    assert L.pm_adf_filter(bogus, other, 640, 480, ctypes.byref(K), 0.15, 0.0, 20, None, None, 0, None) == INV
    assert L.pm_adf_filter(bogus, other, 640, 480, ctypes.byref(K), 0.15, 0.03, -1, None, None, 0, None) == INV
    # aliasing input and output
    assert L.pm_adf_filter(bogus, bogus, 640, 480, ctypes.byref(K), 0.15, 0.03, 20, None, None, 0, None) == INV
    # missing workspace for a multi-pass filter
    assert L.pm_adf_filter(bogus, other, 640, 480, ctypes.byref(K), 0.15, 0.03, 20, None, None, 0, None) == 2
    # normals need K
    assert L.pm_adf_filter(bogus, other, 64, 48, None, 0.15, 0.03, 2, ctypes.c_void_p(0x200000000), None, 0, None) == INV
    # ransac parameter ranges
    ok_ws = ctypes.c_void_p(0x300000000)
    big = 1 << 40
    assert L.pm_ransac_planes(bogus, 640, 480, ctypes.byref(K), other, 64, 0, 0.01, 1, ok_ws, ok_ws, big, None) == INV
    assert L.pm_ransac_planes(bogus, 640, 480, ctypes.byref(K), other, 64, 5000, 0.01, 1, ok_ws, ok_ws, big, None) == INV
    assert L.pm_ransac_planes(bogus, 640, 480, ctypes.byref(K), other, 64, 64, 0.0, 1, ok_ws, ok_ws, big, None) == INV
    assert L.pm_ransac_planes(bogus, 640, 480, ctypes.byref(K), other, -1, 64, 0.01, 1, ok_ws, ok_ws, big, None) == INV
    assert L.pm_ransac_planes(bogus, 640, 480, ctypes.byref(K), other, 64, 64, 0.01, 1, ok_ws, ok_ws, 16, None) == 2
    # misaligned workspace
    assert L.pm_ransac_planes(bogus, 640, 480, ctypes.byref(K), other, 64, 64, 0.01, 1, ok_ws,
                              ctypes.c_void_p(0x300000004), big, None) == 2
    badK = pm.pm_intrinsics(0.0, 385.0, 319.5, 239.5)
    assert L.pm_normals_from_depth(bogus, 640, 480, ctypes.byref(badK), other, None) == INV
    # zero regions is a no-op, not an error
    assert L.pm_ransac_planes(bogus, 640, 480, ctypes.byref(K), other, 0, 64, 0.01, 1, None, None, 0, None) == 0


def test_product_never_imports_oracle():
    pkg = os.path.join(ROOT, "paper_2411_01919_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".c", ".cpp")):
                txt = open(os.path.join(dirpath, f), errors="ignore").read()
                assert "import oracle" not in txt and "from oracle" not in txt and "oracle.h" not in txt, f
                assert "liboracle" not in txt, f


def test_next_features_reject_bad_arguments_before_launch(pm):
    """NEXT-3 polygon calls and the host pipeline's label formats validate on
    the host (no device work)."""
    L = pm._lib
    v = ctypes.c_void_p
    bogus, other, ws = v(0x1000), v(0x100000000), v(0x300000000)
    prm = pm.pm_polygon_params(48, 8192, 256)
    assert L.pm_region_polygons(None, 640, 480, 1, 64, ctypes.byref(prm), bogus, bogus, bogus, ws, ctypes.c_size_t(1 << 40),
                                None) == 1
    bad = pm.pm_polygon_params(48, 8192, 2)                 # < 3 vertices
    assert L.pm_region_polygons(bogus, 640, 480, 1, 64, ctypes.byref(bad), bogus, bogus, bogus, ws,
                                ctypes.c_size_t(1 << 40), None) == 1
    assert L.pm_region_polygons(bogus, 640, 480, 1, 64, ctypes.byref(prm), bogus, bogus, bogus, ws, ctypes.c_size_t(16),
                                None) == 2
    assert L.pm_region_polygons(bogus, 640, 480, 1, 0, ctypes.byref(prm), bogus, bogus, bogus, None, ctypes.c_size_t(0),
                                None) == 0                   # no regions: no-op
    assert L.pm_region_polygons_workspace_bytes(4, 64, 8192) >= 4 * 64 * 8192 * 4
    assert L.pm_rasterize_polygons(bogus, bogus, 2, 640, 480, 1, 64, bogus, ws, ctypes.c_size_t(1 << 20), None) == 1
    assert L.pm_rasterize_polygons(bogus, bogus, 16, 640, 480, 1, 64, bogus, ws, ctypes.c_size_t(8), None) == 2
    K = pm.pm_intrinsics(385.0, 385.0, 319.5, 239.5)
    assert L.pm_lift_polygon_vertices(bogus, bogus, 16, None, 1, 64, ctypes.byref(K), bogus, None) == 1
    # host pipeline: uint8 labels allow at most 255 regions; unknown formats rejected
    big = ctypes.c_size_t(1 << 40)
    args = lambda lf, R: (other, 1, other, lf, 640, 480, 8, 0, ctypes.byref(K), ctypes.c_float(0.15),
                          ctypes.c_float(0.03), 20, R, 64, ctypes.c_float(0.01), ctypes.c_uint64(1), other, None,
                          None, 8, ws, big, None)
    assert L.pm_process_frames_host(*args(pm.LABELS_U8, 256)) == 1
    assert L.pm_process_frames_host(*args(7, 64)) == 1
    assert L.pm_process_frames_host_async(*args(7, 64)) == 1
