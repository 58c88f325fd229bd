#!/usr/bin/env python
"""Time the NEXT-3 polygon glue on the bench workload (C4 frames, 64 balanced
regions per frame): contours + Douglas-Peucker, rasterisation, vertex lifting."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import bench
import paper_2411_01919_b200 as pm
import scenegen

B = int(sys.argv[1]) if len(sys.argv) > 1 else 512
dev = torch.device("cuda", 0)
depth, labels, K = scenegen.stair_stream(0, B, bench.W, bench.H, bench.REGIONS, device=dev)
planes = pm.ransac_planes(depth, K, labels, bench.REGIONS, bench.HYPS, bench.TAU, bench.SEED)
ws = torch.empty(pm._lib.pm_region_polygons_workspace_bytes(B, bench.REGIONS, 8192), dtype=torch.uint8, device=dev)


def timed(fn, reps=5):
    for _ in range(2):
        fn()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        r = fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps, r


t_poly, polys = timed(lambda: pm.region_polygons(labels, bench.REGIONS, 3.0, 8192, 256, workspace=ws))
t_ras, ras = timed(lambda: pm.rasterize_polygons(polys, bench.W, bench.H))
t_lift, X = timed(lambda: pm.lift_polygon_vertices(polys, planes, K))
nv = polys.n_vertices.float()
agree = (ras == labels).float().mean().item()
print(f"frames {B}: contours+DP {t_poly:.3f} ms ({t_poly / B * 1e3:.1f} us/frame), rasterise {t_ras:.3f} ms, "
      f"lift {t_lift:.3f} ms; vertices/polygon mean {nv.mean():.1f} max {nv.max():.0f}; "
      f"max contour {polys.contour_len.max().item()}; rasterised labels == input labels on {agree * 100:.2f}% of pixels")
