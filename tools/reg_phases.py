#!/usr/bin/env python
"""Per-phase SM-cycle breakdown of the register ADF engine (needs the
PM_REG_TIMING variant: tools/build_variant.sh timing -DPM_REG_TIMING):
PMAP_LIB_VARIANT=timing python tools/reg_phases.py [B] [T]"""
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
dev = torch.device("cuda", 0)
depth, labels, K = scenegen.stair_stream(0, B, bench.W, bench.H, bench.REGIONS, device=dev)
out = torch.empty_like(depth)
nrm = torch.empty(B, 3, bench.H, bench.W, device=dev)
ws = torch.empty(pm.adf_workspace_bytes(bench.W, bench.H, B), dtype=torch.uint8, device=dev)
f = lambda: pm.adf_filter(depth, K, bench.LAM, bench.KAPPA, bench.ITERS, iters_per_pass=T, engine=3, out=out,
                          normals_out=nrm, workspace=ws)
f()
torch.cuda.synchronize()
buf = (ctypes.c_ulonglong * 8)()
pm._lib.pm_debug_reg_prof(buf, 1)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
f()
e1.record()
torch.cuda.synchronize()
pm._lib.pm_debug_reg_prof(buf, 1)
names = ["tma wait", "load+scan+sync", "edges+sync", "sweeps", "depth stores", "normals"]
tot = sum(buf[i] for i in range(6))
ms = e0.elapsed_time(e1)
print(f"B={B} T={T}: {ms:.3f} ms; summed CTA cycles {tot:.3e} (= {tot / 1.9e9 / 296 * 1e3:.3f} ms at 2 CTA/SM-equivalent)")
for i, n in enumerate(names):
    print(f"  {n:16s} {buf[i] / tot * 100:5.1f} %  {buf[i]:.3e} cycles")
