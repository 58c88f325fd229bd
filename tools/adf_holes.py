#!/usr/bin/env python
"""ADF+normals stage on 512 C4 frames: hole-free and with 0.1 / 1 / 3 / 6 %
dropout holes: TILED, HOLES and AUTO (which follows the recent calls); each
result compared bit for bit with the register engine (an independent
hole-aware walk)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2411_01919_b200 as pm
import scenegen

B = 512
dev = torch.device("cuda", 0)
d, lab, K = scenegen.stair_stream(0, B, 640, 480, 64, device=dev)
out = torch.empty_like(d)
nrm = torch.empty(B, 3, 480, 640, device=dev)
ws = torch.empty(pm.adf_workspace_bytes(640, 480, B), dtype=torch.uint8, device=dev)
res = {}
for frac, eng in [(f, e) for f in (0.0, 0.001, 0.01, 0.03, 0.06) for e in (pm.ENGINE_TILED, pm.ENGINE_HOLES, pm.ENGINE_AUTO)]:
    x = d.clone()
    if frac:
        for i in range(B):
            x[i] = scenegen.dropout(x[i], frac, 1000 + i, i)
    f = lambda: pm.adf_filter(x, K, 0.15, 0.03, 20, out=out, normals_out=nrm, workspace=ws, engine=eng)
    for _ in range(3):
        f()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(10):
        f()
    e1.record()
    torch.cuda.synchronize()
    res[frac, eng] = e0.elapsed_time(e1) / 10
    ro, rn = pm.adf_filter(x[:32], K, 0.15, 0.03, 20, engine=pm.ENGINE_REG)
    same = torch.equal(out[:32], ro) and torch.equal(nrm[:32].nan_to_num(7.0), rn.nan_to_num(7.0))
    name = {pm.ENGINE_HOLES: "holes", pm.ENGINE_TILED: "tiled", pm.ENGINE_AUTO: "auto"}[eng]
    print(f"{100 * frac:4.1f} % holes, {name}: {res[frac, eng]:.3f} ms per 512 frames  "
          f"({res[frac, eng] / res[0.0, pm.ENGINE_TILED]:.2f}x hole-free tiled)"
          f"  bitwise = register engine: {same}")
