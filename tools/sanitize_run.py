#!/usr/bin/env python
"""Small invocation of every pmap kernel (C1-size frames and a 256x160 frame
for the register engine, both ADF engines and schemes, lambda at the
stability limit, normals, compaction, RANSAC incl. debug/ENUMERATE/
select-error, the host pipeline, segmentation, polygons) for
compute-sanitizer runs (memcheck, racecheck, synccheck, initcheck)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2411_01919_b200 as pm
import scenegen

fr = scenegen.make_config("C1n", holes=0.02)
d, lab, K = fr["depth"].cuda(), fr["labels"].cuda(), fr["K"]
for eng in (pm.ENGINE_TILED, pm.ENGINE_REG, pm.ENGINE_HOLES):
    for scheme in (pm.ADF_ALG1, pm.ADF_DIVERGENCE):
        out, nrm = pm.adf_filter(d, K, 0.15, 0.03, 10, engine=eng, scheme=scheme)
fr2 = scenegen.make_config("C2", W=256, H=160, holes=0.01)
d2 = fr2["depth"].cuda()
for eng in (pm.ENGINE_TILED, pm.ENGINE_REG, pm.ENGINE_HOLES):
    for lam in (0.15, 0.25):
        pm.adf_filter(d2, fr2["K"], lam, 0.03, 9, engine=eng, iters_per_pass=4)
        pm.adf_filter(d2, fr2["K"], lam, 0.03, 9, engine=eng, iters_per_pass=3, normals_mode=pm.NORMALS_AS_PRINTED)
pm.normals_from_depth(d, K)
pm.normals_from_depth(d, K, mode=pm.NORMALS_AS_PRINTED)
pm.ransac_planes(out, K, lab, 4, 64, 0.01, 1, debug=True)
pm.ransac_planes(out, K, lab, 4, 300, 0.01, 1, select=pm.SELECT_ERROR, debug=True)
pm.ransac_planes(out, K, lab, 4, 100, 0.01, 1, select=pm.SELECT_COUNT_EARLY)
pm.ransac_planes(out, K, lab, 4, 100, 0.01, 1, select=pm.SELECT_ERROR_EARLY, debug=True)
pm.ransac_planes(out, K, lab, 4, 1000, 0.01, 1, sampler=pm.SAMPLER_ENUMERATE, debug=True)
ds, ls, K2 = scenegen.stair_stream(0, 3, 128, 96, 16)
pm.process_frames(ds.cuda(), ls.cuda(), K2, 0.15, 0.03, 20, 16, 64, 0.01, 7)
pm.process_frames_host(ds.contiguous(), ls.contiguous(), K2, 0.15, 0.03, 20, 16, 64, 0.01, 7, chunk_frames=2)
# odd W*H: the second frame's points start 8 B off a 16-B boundary (refit bulk
# copies round down / up inside the workspace)
do, lo, K3 = scenegen.stair_stream(0, 3, 333, 251, 16)
pm.process_frames(do.cuda(), lo.cuda(), K3, 0.15, 0.03, 10, 16, 64, 0.01, 7)
# NEXT-2 / NEXT-3 kernels
_, n2 = pm.adf_filter(d2, fr2["K"], 0.15, 0.03, 20)
labels, nreg, _ = pm.segment_regions(n2, 30, 90, 100, 64, edges=True)
polys = pm.region_polygons(labels, 64)
pm.rasterize_polygons(polys, 256, 160)
pl = pm.ransac_planes(d2, fr2["K"], labels, 64, 64, 0.01, 3)
# many small regions: the warp-per-segment scoring kernel (count-only)
v, u = torch.meshgrid(torch.arange(160, device="cuda"), torch.arange(256, device="cuda"), indexing="ij")
grid = ((v // 8) * 32 + u // 8).to(torch.int32)
pm.ransac_planes(d2, fr2["K"], grid, 640, 64, 0.01, 3, debug="counts")
pm.lift_polygon_vertices(polys, pl, fr2["K"])
torch.cuda.synchronize()
print("sanitize run ok")
