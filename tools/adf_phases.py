#!/usr/bin/env python
"""Per-phase SM-cycle breakdown of the tiled ADF engine (needs the
PM_ADF_TIMING variant: tools/build_variant.sh atiming -DPM_ADF_TIMING):
PMAP_LIB_VARIANT=atiming python tools/adf_phases.py [B] [T] [holes] [engine]"""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import bench
import paper_2411_01919_b200 as pm
import scenegen

B = int(sys.argv[1]) if len(sys.argv) > 1 else 512
T = int(sys.argv[2]) if len(sys.argv) > 2 else 4
holes = float(sys.argv[3]) if len(sys.argv) > 3 else 0.0
engine = int(sys.argv[4]) if len(sys.argv) > 4 else 1
dev = torch.device("cuda", 0)
depth, labels, K = scenegen.stair_stream(0, B, bench.W, bench.H, bench.REGIONS, device=dev)
if holes > 0:
    for i in range(B):
        depth[i] = scenegen.dropout(depth[i], holes, 1000 + i, i)
out = torch.empty_like(depth)
nrm = torch.empty(B, 3, bench.H, bench.W, device=dev)
ws = torch.empty(pm.adf_workspace_bytes(bench.W, bench.H, B), dtype=torch.uint8, device=dev)
f = lambda: pm.adf_filter(depth, K, bench.LAM, bench.KAPPA, bench.ITERS, iters_per_pass=T, engine=engine, out=out,
                          normals_out=nrm, workspace=ws)
f()
torch.cuda.synchronize()
buf = (ctypes.c_ulonglong * 8)()
pm._lib.pm_debug_adf_prof(buf, 1)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
f()
e1.record()
torch.cuda.synchronize()
pm._lib.pm_debug_adf_prof(buf, 1)
ms = e0.elapsed_time(e1)
tot = sum(buf[i] for i in range(8))
print(f"B={B} T={T} holes={holes} engine={engine}: {ms:.3f} ms; summed CTA cycles {tot:.3e}")
for i, n in enumerate(["plain load+scan", "plain sweeps", "plain epilogue", "-", "fused load+scan", "fused sweeps",
                       "fused epilogue (stores+normals)"]):
    if n != "-":
        print(f"  {n:32s} {buf[i] / tot * 100:5.1f} %  {buf[i]:.3e}")
