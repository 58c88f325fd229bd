#!/usr/bin/env python
"""ADF+normals stage over 512 C4 frames issued as chunks of C frames (same
stream): does keeping a chunk's intermediate passes in L2 pay?"""
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
for C in (512, 256, 128, 64, 32, 16):
    ws = torch.empty(pm.adf_workspace_bytes(bench.W, bench.H, C), dtype=torch.uint8, device=dev)

    def run():
        for s in range(0, B, C):
            pm.adf_filter(depth[s:s + C], K, bench.LAM, bench.KAPPA, bench.ITERS, out=out[s:s + C],
                          normals_out=nrm[s:s + C], workspace=ws, engine=int(os.environ.get("ENG", "1")))
    for _ in range(3):
        run()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(10):
        run()
    e1.record()
    torch.cuda.synchronize()
    print(f"chunk {C:4d}: {e0.elapsed_time(e1) / 10:.3f} ms per 512 frames")
