#!/usr/bin/env python
"""Run the ADF+normals stage on the bench workload (for ncu): adf_only.py B engine T reps."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import bench
import paper_2411_01919_b200 as pm
import scenegen

B, eng, T, reps = (int(a) for a in (sys.argv[1:] + ["64", "3", "4", "2"][len(sys.argv) - 1:]))
holes = float(os.environ.get("PM_HOLES", "0"))
dev = torch.device("cuda", 0)
depth, labels, K = scenegen.stair_stream(0, B, bench.W, bench.H, bench.REGIONS, device=dev)
if holes > 0:
    depth = scenegen.dropout(depth, holes, 123, 0)
out = torch.empty_like(depth)
nrm = torch.empty(B, 3, bench.H, bench.W, device=dev)
ws = torch.empty(pm.adf_workspace_bytes(bench.W, bench.H, B), dtype=torch.uint8, device=dev)
for _ in range(reps):
    pm.adf_filter(depth, K, bench.LAM, bench.KAPPA, bench.ITERS, iters_per_pass=T, engine=eng, out=out,
                  normals_out=nrm, workspace=ws)
torch.cuda.synchronize()
print("ok")
