#!/usr/bin/env python
"""Minimal driver for ncu captures: the bench workload (C4 stream frames,
pm_process_frames) run `--reps` times on `--frames` resident frames, nothing
else.  Use with ncu -k regex:"adf_|compact_|ransac_"."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import bench
import paper_2411_01919_b200 as pm
import scenegen

ap = argparse.ArgumentParser()
ap.add_argument("--frames", type=int, default=64)
ap.add_argument("--reps", type=int, default=2)
a = ap.parse_args()
dev = torch.device("cuda", 0)
depth, labels, K = scenegen.stair_stream(0, a.frames, bench.W, bench.H, bench.REGIONS, device=dev)
ws = torch.empty(pm.pipeline_workspace_bytes(bench.W, bench.H, bench.REGIONS, bench.HYPS, a.frames),
                 dtype=torch.uint8, device=dev)
for _ in range(a.reps):
    pm.process_frames(depth, labels, K, bench.LAM, bench.KAPPA, bench.ITERS, bench.REGIONS, bench.HYPS, bench.TAU,
                      bench.SEED, workspace=ws)
torch.cuda.synchronize()
print("ok")
