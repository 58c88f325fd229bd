#!/usr/bin/env python
"""Time ransac_planes on the bench workload (filtered frames) -> per-stage ms."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import bench
import paper_2411_01919_b200 as pm
import scenegen

B = int(sys.argv[1]) if len(sys.argv) > 1 else 512
H_hyp = int(sys.argv[2]) if len(sys.argv) > 2 else bench.HYPS
dev = torch.device("cuda", 0)
depth, labels, K = scenegen.stair_stream(0, B, bench.W, bench.H, bench.REGIONS, device=dev)
filt, _ = pm.adf_filter(depth, K, bench.LAM, bench.KAPPA, bench.ITERS, normals=False)
ws = torch.empty(pm.ransac_workspace_bytes(bench.W, bench.H, bench.REGIONS, H_hyp, B), dtype=torch.uint8, device=dev)
out = torch.empty(B, bench.REGIONS, pm.PLANE_WORDS, dtype=torch.int32, device=dev)
f = lambda: pm.ransac_planes(filt, K, labels, bench.REGIONS, H_hyp, bench.TAU, bench.SEED, out=out, workspace=ws)
for _ in range(3):
    f()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10):
    f()
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 10
print(f"lanes={os.environ.get('PM_SCORE_LANES', 'auto')} H={H_hyp} ransac {ms:.3f} ms / {B} frames = {ms * 1e3 / B:.2f} us/frame; "
      f"status ok {float((pm.Planes(out).status == 0).float().mean()):.3f} checksum {int(out.sum())}")
