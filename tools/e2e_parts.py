#!/usr/bin/env python
"""Where the host-fed (e2e) step goes: H2D alone (pinned -> device, 64-frame
chunks on one stream), the kernels alone on 64-frame device chunks, and the
pipeline (pm_process_frames_host) -- 512 C4 frames, run-length labels."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import bench
import paper_2411_01919_b200 as pm
import scenegen

B, C = 512, int(sys.argv[1]) if len(sys.argv) > 1 else 64
dev = torch.device("cuda", 0)
d, lab, K = scenegen.stair_stream(0, B, 640, 480, 64, device=dev)
h_mm = torch.round(d.double() * 1000).clamp(0, 65535).to(torch.int32).to(torch.uint16).cpu().pin_memory()
runs = pm.encode_label_runs(lab.cpu()).pin_memory()
dev_mm = torch.empty(C, 480, 640, dtype=torch.uint16, device=dev)


def timeit(f, n=5):
    f()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n):
        f()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n


def h2d():
    for s in range(0, B, C):
        dev_mm.copy_(h_mm[s:s + C], non_blocking=True)


t_h2d = timeit(h2d)
dm = d.clone()
ws = torch.empty(pm.pipeline_workspace_bytes(640, 480, 64, 64, C), dtype=torch.uint8, device=dev)
do = torch.empty(C, 480, 640, device=dev)
nr = torch.empty(C, 3, 480, 640, device=dev)
pl = torch.empty(C, 64, 12, dtype=torch.int32, device=dev)


def kern():
    for s in range(0, B, C):
        pm.process_frames(dm[s:s + C], lab[s:s + C], K, bench.LAM, bench.KAPPA, 20, 64, 64, bench.TAU, bench.SEED,
                          first_frame_id=s, depth_out=do, normals_out=nr, planes_out=pl, workspace=ws)


t_k = timeit(kern)
arena = torch.empty(pm.host_pipeline_arena_bytes(640, 480, 64, 64, C, pm.DEPTH_U16_MM, pm.LABELS_RUNS),
                    dtype=torch.uint8, device=dev)
hp = torch.empty(B, 64, 12, dtype=torch.int32).pin_memory()
t_p = timeit(lambda: pm.process_frames_host(h_mm, runs, K, bench.LAM, bench.KAPPA, 20, 64, 64, bench.TAU, bench.SEED,
                                            chunk_frames=C, planes_out=hp, arena=arena, device=dev))
print(f"chunk {C}: H2D depth alone {t_h2d:.2f} ms ({h_mm.numel() * 2 / t_h2d / 1e6:.1f} GB/s); kernels alone "
      f"{t_k:.2f} ms; pipeline {t_p:.2f} ms ({B / t_p * 1e3:.0f} frames/s)")
