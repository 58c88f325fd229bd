#!/usr/bin/env python
"""Time segment_regions on the bench workload's normals (512 frames)."""
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
d, nrm = pm.adf_filter(depth, K, bench.LAM, bench.KAPPA, bench.ITERS)
ws = torch.empty(pm.segment_workspace_bytes(bench.W, bench.H, B, 300), dtype=torch.uint8, device=dev)
f = lambda: pm.segment_regions(nrm, 30, 90, 300, 64, workspace=ws)
for _ in range(3):
    lab, nreg, _ = f()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10):
    f()
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 10
print(f"segment_regions {ms:.3f} ms / {B} frames = {ms * 1e3 / B:.2f} us/frame; regions/frame "
      f"mean {nreg.float().mean():.1f} min {int(nreg.min())} max {int(nreg.max())}")
