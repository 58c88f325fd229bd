#!/usr/bin/env python
"""Does running the ADF of one half of the batch next to the RANSAC of the
other half (two streams) beat the serial pipeline?  Times, on the bench's
512 C4 frames: (a) one pm_process_frames call; (b) two halves on two streams,
the second half's ADF started when the first half's ADF ends (so it runs
beside the first half's RANSAC); (c) n parts round-robin on two streams.
Results must stay bitwise equal to (a)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import bench
import paper_2411_01919_b200 as pm
import scenegen

B, W, H, R, HYP = 512, bench.W, bench.H, bench.REGIONS, bench.HYPS
dev = torch.device("cuda", 0)
depth, labels, K = scenegen.stair_stream(0, B, W, H, R, device=dev)
d_out = torch.empty_like(depth)
nrm = torch.empty(B, 3, H, W, device=dev)
planes = torch.empty(B, R, pm.PLANE_WORDS, dtype=torch.int32, device=dev)
ws_full = torch.empty(pm.pipeline_workspace_bytes(W, H, R, HYP, B), dtype=torch.uint8, device=dev)


def full():
    pm.process_frames(depth, labels, K, bench.LAM, bench.KAPPA, bench.ITERS, R, HYP, bench.TAU, bench.SEED,
                      depth_out=d_out, normals_out=nrm, planes_out=planes, workspace=ws_full)


def timed(f, n=10):
    for _ in range(3):
        f()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n):
        f()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n


def make_parts(n_parts, prio):
    step = B // n_parts
    streams = [torch.cuda.Stream(device=dev, priority=prio[0]), torch.cuda.Stream(device=dev, priority=prio[1])]
    adf_ws = [torch.empty(pm.adf_workspace_bytes(W, H, step), dtype=torch.uint8, device=dev) for _ in range(2)]
    rs_ws = [torch.empty(pm.ransac_workspace_bytes(W, H, R, HYP, step), dtype=torch.uint8, device=dev)
             for _ in range(2)]

    def run():
        main = torch.cuda.current_stream()
        start = torch.cuda.Event()
        start.record(main)
        prev_adf = None
        ends = []
        for i in range(n_parts):
            s = streams[i % 2]
            sl = slice(i * step, (i + 1) * step)
            with torch.cuda.stream(s):
                s.wait_event(start)
                if prev_adf is not None:
                    s.wait_event(prev_adf)
                pm.adf_filter(depth[sl], K, bench.LAM, bench.KAPPA, bench.ITERS, out=d_out[sl], normals_out=nrm[sl],
                              workspace=adf_ws[i % 2])
                prev_adf = torch.cuda.Event()
                prev_adf.record(s)
                pm.ransac_planes(d_out[sl], K, labels[sl], R, HYP, bench.TAU, bench.SEED, first_frame_id=i * step,
                                 out=planes[sl], workspace=rs_ws[i % 2])
                e = torch.cuda.Event()
                e.record(s)
                ends.append(e)
        for e in ends:
            main.wait_event(e)
    return run


t_full = timed(full)
ref = (d_out.clone(), nrm.clone(), planes.clone())
print(f"serial pm_process_frames: {t_full:.3f} ms  ({B / t_full * 1e3:.0f} frames/s)")
for n_parts in (2, 4, 8):
    for prio in ((0, 0), (-1, 0), (0, -1)):
        d_out.zero_(); nrm.zero_(); planes.zero_()
        t = timed(make_parts(n_parts, prio))
        same = torch.equal(d_out, ref[0]) and torch.equal(nrm, ref[1]) and torch.equal(planes, ref[2])
        print(f"{n_parts} parts on 2 streams, priorities {prio}: {t:.3f} ms ({B / t * 1e3:.0f} frames/s) "
              f"bitwise_same={same}")
