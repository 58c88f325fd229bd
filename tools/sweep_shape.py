#!/usr/bin/env python
"""The paper's fig:ex2a shape claims (SURVEY §8(d) extra sweeps):
per-frame time of the whole path (pm_process_frames) vs resolution at N=10,
H=10 and vs region count at 640x480 (N=20, H=64).  The paper runs polygons
sequentially, so its time grows linearly with the region count; the batched
design here should be about flat (evaluations = H x labelled pixels).  Each
point also reports the ADF+normals stage's FP32 fraction and the scoring
kernel's issue-bound fraction (bench.py's §8(d) definitions, at the clock
given as the first argument, MHz; default 1965)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import bench
import paper_2411_01919_b200 as pm
import scenegen

CLK = float(sys.argv[1]) if len(sys.argv) > 1 else 1965.0

dev = torch.device("cuda", 0)


def timed(B, W, H, R, N, NH, reps=5):
    # 4 distinct frames tiled to B (label generation with the balanced-region
    # guard is slow for R ~ 1000 on the host)
    d4, lab4, K = scenegen.stair_stream(0, 4, W, H, R, device="cpu")
    d = d4.repeat((B + 3) // 4, 1, 1)[:B].contiguous().to(dev)
    lab = lab4.repeat((B + 3) // 4, 1, 1)[:B].contiguous().to(dev)
    ws = torch.empty(pm.pipeline_workspace_bytes(W, H, R, NH, B), dtype=torch.uint8, device=dev)
    dout = torch.empty_like(d)
    nrm = torch.empty(B, 3, H, W, device=dev)
    pl = torch.empty(B, R, pm.PLANE_WORDS, dtype=torch.int32, device=dev)
    f = lambda: pm.process_frames(d, lab, K, 0.15, 0.03, N, R, NH, 0.01, 0x1919, depth_out=dout, normals_out=nrm,
                                  planes_out=pl, workspace=ws)
    for _ in range(2):
        f()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        f()
    e1.record()
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) / reps / B * 1e3   # us per frame
    st = bench.stage_times(pm, d, lab, K, N, R, NH, 0, ws, dout, nrm, pl, reps=3)
    adf_frac = (11 * N + bench.NORMAL_OPS_PER_PIX) * W * H * B / (st["adf_normals"] * 1e-3) / bench._alu_peak(CLK)
    evals = NH * bench._labelled(d, lab, R)
    score_frac = evals / (st["score"] * 1e-3) / bench._score_issue_peak(CLK)
    return f"{us:8.2f} us/frame   ADF FP32 frac {adf_frac:.3f}   score issue frac {score_frac:.3f}   " \
           f"(ADF {st['adf_normals'] / B * 1e3:.2f} us/frame, RANSAC {st['ransac'] / B * 1e3:.2f} us/frame)"


print("resolution sweep (N=10, H=10, R=64):")
for W, H, B in ((320, 240, 1024), (640, 480, 512), (1280, 720, 128)):
    print(f"  {W}x{H}: {timed(B, W, H, 64, 10, 10)}")
print("region-count sweep (640x480, N=20, H=64):")
for R in (4, 16, 64, 256, 1024):  # noqa: E501
    print(f"  R={R:5d}: {timed(256, 640, 480, R, 20, 64)}")
