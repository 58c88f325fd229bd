#!/usr/bin/env python
"""Time the adf_filter stage (bench workload) for several sweeps-per-pass T."""
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
out = torch.empty_like(depth)
nrm = torch.empty(B, 3, bench.H, bench.W, device=dev)
ws = torch.empty(pm.adf_workspace_bytes(bench.W, bench.H, B), dtype=torch.uint8, device=dev)
ref = None
ENG = {1: "tiled", 3: "reg"}
cfgs = [(1, 4), (1, 5), (3, 4), (3, 5)]
if len(sys.argv) > 2:
    cfgs = [tuple(map(int, c.split(":"))) for c in sys.argv[2].split(",")]
for eng, T in cfgs:
    f = lambda: pm.adf_filter(depth, K, bench.LAM, bench.KAPPA, bench.ITERS, iters_per_pass=T, engine=eng, out=out,
                              normals_out=nrm, workspace=ws)
    for _ in range(3):
        f()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        f()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 10
    if ref is None:
        ref = out.clone()
    same = torch.equal(out, ref)
    print(f"engine={ENG[eng]:6s} T={T:2d} {ms:7.3f} ms/stage  {ms * 1e3 / B:6.2f} us/frame  "
          f"{bench.ITERS * bench.W * bench.H * B / ms / 1e9:6.2f} Gpix-iter/s  bitwise_same={same}")
