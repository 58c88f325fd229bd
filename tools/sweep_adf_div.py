#!/usr/bin/env python
"""ADF stage time, Alg. 1 vs the divergence-form scheme (NEXT-1), bench frames."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import bench
import paper_2411_01919_b200 as pm
import scenegen

B = 512
dev = torch.device("cuda", 0)
depth, labels, K = scenegen.stair_stream(0, B, bench.W, bench.H, bench.REGIONS, device=dev)
out = torch.empty_like(depth)
nrm = torch.empty(B, 3, bench.H, bench.W, device=dev)
ws = torch.empty(pm.adf_workspace_bytes(bench.W, bench.H, B), dtype=torch.uint8, device=dev)
for name, sch in (("alg1", pm.ADF_ALG1), ("divergence", pm.ADF_DIVERGENCE)):
    f = lambda: pm.adf_filter(depth, K, bench.LAM, bench.KAPPA, bench.ITERS, out=out, normals_out=nrm, workspace=ws,
                              scheme=sch)
    for _ in range(3):
        f()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        f()
    e1.record()
    torch.cuda.synchronize()
    print(f"{name}: ADF+normals {e0.elapsed_time(e1) / 5:.3f} ms / {B} frames")
