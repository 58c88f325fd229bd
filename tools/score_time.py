#!/usr/bin/env python
"""RANSAC per-kernel times (stage events) on the bench workload (512 C4
frames, filtered depth): python tools/score_time.py [frames]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import bench
import paper_2411_01919_b200 as pm
import scenegen

B = int(sys.argv[1]) if len(sys.argv) > 1 else 512
dev = torch.device("cuda", 0)
d, lab, K = scenegen.stair_stream(0, B, 640, 480, 64, device=dev)
out = torch.empty_like(d)
nrm = torch.empty(B, 3, 480, 640, device=dev)
ws = torch.empty(pm.pipeline_workspace_bytes(640, 480, 64, 64, B), dtype=torch.uint8, device=dev)
pl = torch.empty(B, 64, 12, dtype=torch.int32, device=dev)
st = bench.stage_times(pm, d, lab, K, 20, 64, 64, 0, ws, out, nrm, pl, reps=5)
print({k: round(v, 4) for k, v in st.items()})
