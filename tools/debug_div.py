"""Locate bitwise differences of the divergence-scheme ADF between blockings."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2411_01919_b200 as pm
import scenegen

fr = scenegen.make_config(sys.argv[1] if len(sys.argv) > 1 else "C2")
d = fr["depth"].cuda()
print("invalid px:", int((fr["depth"] <= 0).sum()), "shape", tuple(d.shape))
outs = {}
for sch in (pm.ADF_ALG1, pm.ADF_DIVERGENCE):
    for T in (1, 2, 3, 4, 5):
        for nrm in (False, True):
            o, _ = pm.adf_filter(d, fr["K"], fr["lam"], fr["kappa"], fr["iters"], iters_per_pass=T, scheme=sch,
                                 normals=nrm)
            outs[(sch, T, nrm)] = o.cpu().numpy()
    o, _ = pm.adf_filter(d, fr["K"], fr["lam"], fr["kappa"], fr["iters"], iters_per_pass=4, scheme=sch,
                         normals=False, engine=pm.ENGINE_REG)
    outs[(sch, "stream")] = o.cpu().numpy()
    ref = outs[(sch, "stream")]
    for k, v in outs.items():
        if k[0] != sch:
            continue
        diff = np.nonzero(v != ref)
        print(sch, k, "ndiff", len(diff[0]), "rows", np.unique(diff[0])[:10], "cols", np.unique(diff[1])[:20],
              "maxabs", float(np.abs(v - ref).max()) if len(diff[0]) else 0)
