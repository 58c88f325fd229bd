#!/usr/bin/env python
"""One adf_filter call (bench workload, 512 C4 frames) per sweeps-per-pass T
given on the command line -- for an ncu launch list of per-pass DRAM
throughput (tools/sweep_adf.py times the same configurations without ncu)."""
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
for T in map(int, sys.argv[1].split(",")):
    pm.adf_filter(depth, K, bench.LAM, bench.KAPPA, bench.ITERS, iters_per_pass=T, out=out, normals_out=nrm,
                  workspace=ws)
torch.cuda.synchronize()
