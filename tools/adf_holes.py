#!/usr/bin/env python
"""ADF+normals stage on 512 C4 frames, hole-free and with 1 % dropout holes."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2411_01919_b200 as pm
import scenegen

B = 512
dev = torch.device("cuda", 0)
d, lab, K = scenegen.stair_stream(0, B, 640, 480, 64, device=dev)
dh = d.clone()
for i in range(B):
    dh[i] = scenegen.dropout(dh[i], 0.01, 1000 + i, i)
out = torch.empty_like(d)
nrm = torch.empty(B, 3, 480, 640, device=dev)
ws = torch.empty(pm.adf_workspace_bytes(640, 480, B), dtype=torch.uint8, device=dev)
res = {}
for name, x in (("hole-free", d), ("1% holes", dh)):
    f = lambda: pm.adf_filter(x, K, 0.15, 0.03, 20, out=out, normals_out=nrm, workspace=ws)
    for _ in range(3):
        f()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(10):
        f()
    e1.record()
    torch.cuda.synchronize()
    res[name] = e0.elapsed_time(e1) / 10
    print(f"{name:10s}: {res[name]:.3f} ms per 512 frames")
print(f"ratio holes / hole-free: {res['1% holes'] / res['hole-free']:.2f}")
