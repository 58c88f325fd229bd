#!/usr/bin/env python
"""Benchmark of the arXiv 2411.01919 hot path on B200 (BASELINE.json metric).

Workload (BASELINE.json configs[3], "C4"): a stream of distinct synthetic
640x480 D435-style noisy descending-staircase frames (scenegen G-STAIR,
DESIGN.md §4), N = 20 ADF iterations (lambda 0.15, kappa 0.03 m) with the
normal image fused into the last pass, then RANSAC over 64 balanced regions
per frame x 64 hypotheses (tau 0.01 m) on the filtered depth.  One step = one
pass of the whole path over this rank's batch of frames (frames_per_rank),
all resident in HBM; ranks process disjoint frames of the stream (frame ids
rank * frames_per_rank + i): weak scaling, no data-path collective, a final
NCCL gather of the plane tables only in the multi-GPU run.

Arms:
  default            the CUDA path through the C ABI (pm_process_frames)
  --impl reference   the oracle (oracle/, plain single-threaded C per frame)
                     on this box's host cores, same workload and metric.
Prints ONE JSON line on rank 0.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

METRIC = "640x480 frames/sec per B200 and at 8 GPUs; ADF+normal achieved HBM GB/s vs peak"
W, H = 640, 480
ITERS, REGIONS, HYPS = 20, 64, 64
LAM, KAPPA, TAU, SEED = 0.15, 0.03, 0.01, 0x1919
# algorithmic bytes of the fused ADF+normals stage per pixel: read depth 4 B,
# write filtered depth 4 B, write normals 12 B
ADF_ALG_BYTES_PX = 20
# FP32 lane-ops of one Alg. 1 sweep at one pixel:
# 2gx, 2gy, gy^2, gx^2+, exponent FFMA, ex2, three adds and an FFMA for the
# Laplacian, the update FFMA
ADF_OPS_PER_PIX_ITER = 11
# FP32 lane-ops of the Sobel + normal stage per pixel (~22 FP32 + 1 rsqrt)
NORMAL_OPS_PER_PIX = 22
# one RANSAC point-hypothesis evaluation: 3 FFMA (n.p + d), compare, count =
# 5 issue slots; the issue bound is 148 SMs x 4 schedulers x
# 32 lanes x clock / 5 evaluations per second
RANSAC_ISSUE_PER_EVAL = 5
WORKLOAD = ("C4 (BASELINE.json configs[3]): stream of distinct 640x480 D435-noise G-STAIR frames; ADF N=20 "
            "(lambda 0.15, kappa 0.03 m) + fused normals, RANSAC 64 regions x 64 hypotheses (tau 0.01 m) on the "
            "filtered depth")


def _ncu_traffic():
    """DRAM bytes (read + write) of one ADF+normals stage on this workload,
    from the committed ncu capture profiles/adf_traffic.json (same unit as
    `achieved`: the whole stage), or None."""
    p = os.path.join(ROOT, "profiles", "adf_traffic.json")
    if os.path.exists(p):
        with open(p) as f:
            return json.load(f).get("bytes_per_stage")
    return None


def _peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            j = json.load(f)
        return float(j["hbm_gbs"]), "measured (MEASURED_PEAKS.json)"
    return 6650.0, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """Samples SM clock and throttle reasons with NVML during the timed region."""

    REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
               0x10: "sync_boost", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
               0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting"}

    def __init__(self, index: int, period_s: float = 0.002):
        # NVML enumerates physical GPUs; honour CUDA_VISIBLE_DEVICES when it is a list of indices
        vis = os.environ.get("CUDA_VISIBLE_DEVICES", "")
        try:
            ids = [int(x) for x in vis.split(",") if x.strip() != ""]
            if ids and index < len(ids):
                index = ids[index]
        except ValueError:
            pass
        self.index, self.period = index, period_s
        self.samples, self.reasons = [], set()
        self._stop = threading.Event()
        self._t = None
        self.max_mhz = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self._nv = pynvml
            self._h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self._h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self._nv = None

    def _run(self):
        nv = self._nv
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self._h, nv.NVML_CLOCK_SM))
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(self._h)
                for bit, name in self.REASONS.items():
                    if r & bit and name != "gpu_idle":
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(self.period)

    def __enter__(self):
        if self._nv is not None:
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._t:
            self._t.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["unavailable"]}
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


# --------------------------------------------------------------------------- sharding
def shard(rank: int, frames_per_rank: int):
    """Frames of the C4 stream owned by `rank`: [rank * B, (rank + 1) * B).
    The RNG is keyed by the global frame id, so every sharding gives the
    same per-frame results (weak scaling, no data-path collective)."""
    return rank * frames_per_rank, frames_per_rank


def gather_tables(t, world: int, rank: int):
    """Gather every rank's plane table to rank 0 (the only collective of the
    path); returns the concatenation on rank 0, else None."""
    import torch
    import torch.distributed as dist
    if world == 1:
        return t
    parts = [torch.empty_like(t) for _ in range(world)] if rank == 0 else None
    dist.gather(t, parts, dst=0)
    return torch.cat(parts) if rank == 0 else None


# --------------------------------------------------------------------------- oracle arm
def _oracle_frame(depth_np, labels_np, K, frame_id):
    import oracle
    d = oracle.adf(depth_np, LAM, KAPPA, ITERS)
    oracle.normals(d, K)
    oracle.ransac(d, labels_np, K, REGIONS, HYPS, TAU, SEED, frame_id=frame_id)


def _cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


def _cpu_cores():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def _oracle_throughput(frames, K, first_frame, cores):
    """Run the oracle over `frames` [(depth, labels)] on `cores` threads (the C
    calls release the GIL); returns (frames/s, wall seconds)."""
    from concurrent.futures import ThreadPoolExecutor
    t0 = time.perf_counter()
    with ThreadPoolExecutor(max_workers=cores) as ex:
        list(ex.map(lambda i: _oracle_frame(frames[i][0], frames[i][1], K, first_frame + i), range(len(frames))))
    dt = time.perf_counter() - t0
    return len(frames) / dt, dt


def _cpu_sample(n, first_frame):
    import scenegen
    d, lab, K = scenegen.stair_stream(first_frame, n, W, H, REGIONS, device="cpu")
    return [(d[i].numpy(), lab[i].numpy()) for i in range(n)], K


def run_reference(args, rank, world):
    if rank != 0:
        return 0
    import oracle
    oracle.build()
    cores = _cpu_cores()
    frames, K = _cpu_sample(cores, 0)
    for _ in range(args.warmup):
        _oracle_throughput(frames, K, 0, cores)
    times = []
    for _ in range(args.steps):
        _, dt = _oracle_throughput(frames, K, 0, cores)
        times.append(dt)
    total = sum(times)
    value = cores * args.steps / total
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "frames/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * total / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64+f32",
        "data": "synthetic",
        "config": {"workload": WORKLOAD, "frames_per_step": cores,
                   "sample": f"{cores} frames of the same stream per step (one per host core)"},
        "cpu_baseline": {"value": value, "unit": "frames/s", "cores": cores, "kind": "oracle",
                         "sample": f"{cores} frames per step (one per core), {args.steps} timed steps",
                         "cpu_model": _cpu_model()},
        "e2e": {"value": value, "unit": "frames/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# --------------------------------------------------------------------------- CUDA arm
def _events(n):
    import torch
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(n)]
    for e in ev:          # materialise the CUDA events (created lazily on first record)
        e.record()
    return ev


def _alu_peak(clk_mhz):
    """FP32 lane-op peak: 148 SMs x 128 lanes x SM clock (B200_PROFILING.md unit counts)."""
    return 148 * 128 * clk_mhz * 1e6


def _score_issue_peak(clk_mhz):
    """RANSAC scoring issue bound: 148 SMs x 4 schedulers x 32
    lanes x clock / 5 issue slots per point-hypothesis evaluation."""
    return 148 * 4 * 32 * clk_mhz * 1e6 / RANSAC_ISSUE_PER_EVAL


def stage_times(pm, depth, labels, K, iters, R, H_, first, ws, depth_out, normals, planes, lam=LAM, reps=5):
    """Median per-stage device times (ms) of one batch, in the bench's launch
    configuration on the launch stream: the ADF+normals stage (adf_filter),
    and inside ransac_planes the compaction, hypotheses, scoring (the
    dominant RANSAC kernel, its own events), selection + refit, plane table."""
    import torch
    out = {"adf_normals": [], "ransac": [], "compaction": [], "hypotheses": [], "score": [], "refit": []}
    e0, e1 = _events(2)
    ev = _events(pm.RANSAC_STAGE_EVENTS)
    for _ in range(reps):
        e0.record()
        pm.adf_filter(depth, K, lam, KAPPA, iters, normals=True, out=depth_out, normals_out=normals, workspace=ws)
        e1.record()
        pm.ransac_planes(depth_out, K, labels, R, H_, TAU, SEED, first_frame_id=first, out=planes, workspace=ws,
                         stage_events=ev)
        torch.cuda.synchronize()
        out["adf_normals"].append(e0.elapsed_time(e1))
        out["ransac"].append(ev[0].elapsed_time(ev[5]))
        out["compaction"].append(ev[0].elapsed_time(ev[1]))
        out["hypotheses"].append(ev[1].elapsed_time(ev[2]))
        out["score"].append(ev[2].elapsed_time(ev[3]))
        out["refit"].append(ev[3].elapsed_time(ev[4]))
    return {k: statistics.median(v) for k, v in out.items()}


def rooflines(W_, H_, B, iters, n_hyp, labelled_px, st, clk_mhz, hbm_peak, traffic=None):
    """ADF+normals stage: FP32 lane-ops (11 per pixel-iteration
    + 22 per pixel for the normals) / stage time vs the FP32 peak, and its HBM
    view (20 B/px algorithmic); RANSAC scoring: evaluations / score-kernel
    time vs the §8(d) issue bound."""
    px = W_ * H_ * B
    adf_t = st["adf_normals"] / 1e3
    ops = (iters * ADF_OPS_PER_PIX_ITER + NORMAL_OPS_PER_PIX) * px
    alu = ops / adf_t
    hbm = ADF_ALG_BYTES_PX * px / adf_t / 1e9
    evals = n_hyp * labelled_px
    ev_s = evals / (st["score"] / 1e3)
    return ({"bound": "alu", "kernel": "adf_pass_kernel (ADF+normals stage, last pass fused with the normals)",
             "achieved": alu / 1e12, "peak": _alu_peak(clk_mhz) / 1e12, "unit": "T FP32 lane-op/s",
             "frac": alu / _alu_peak(clk_mhz), "traffic": traffic,
             "alg_ops_per_pixel": iters * ADF_OPS_PER_PIX_ITER + NORMAL_OPS_PER_PIX,
             "peak_source": "148 SMs x 128 FP32 lanes x SM clock (B200_PROFILING.md)",
             "stage_ms": st["adf_normals"],
             "hbm": {"achieved": hbm, "peak": hbm_peak, "unit": "GB/s", "frac": hbm / hbm_peak,
                     "alg_bytes_per_px": ADF_ALG_BYTES_PX}},
            {"bound": "issue", "kernel": "ransac_score_kernel (Alg. 2 l.9-13), its own CUDA-event time",
             "achieved": ev_s / 1e12, "peak": _score_issue_peak(clk_mhz) / 1e12, "unit": "T evals/s",
             "frac": ev_s / _score_issue_peak(clk_mhz), "evals": evals, "score_ms": st["score"],
             "issue_slots_per_eval": RANSAC_ISSUE_PER_EVAL,
             "stage_ms": {k: st[k] for k in ("ransac", "compaction", "hypotheses", "score", "refit")}})


def _labelled(depth, labels, R):
    import torch
    v = (depth > 0) & torch.isfinite(depth) & (labels >= 0) & (labels < R)
    return int(v.sum().item())


def _time_pipeline(pm, depth, labels, K, iters, R, H_, first, steps, warmup, bufs):
    import torch
    d_out, nrm, planes, ws = bufs
    f = lambda: pm.process_frames(depth, labels, K, LAM, KAPPA, iters, R, H_, TAU, SEED, first_frame_id=first,
                                  depth_out=d_out, normals_out=nrm, planes_out=planes, workspace=ws)
    for _ in range(warmup):
        f()
    torch.cuda.synchronize()
    e0, e1 = _events(2)
    e0.record()
    for _ in range(steps):
        f()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / steps


def extra_configs(pm, dev, clk_mhz, hbm_peak):
    """The other BASELINE.json configs and the paper's per-frame context, on
    this GPU (bounded: ~1-2 s each).  Every number is device time with CUDA
    events on the launch stream, inputs resident in HBM."""
    import torch
    import scenegen
    res = {}

    def bufs(B, H, W, R, H_):
        return (torch.empty(B, H, W, device=dev), torch.empty(B, 3, H, W, device=dev),
                torch.empty(B, R, pm.PLANE_WORDS, dtype=torch.int32, device=dev),
                torch.empty(pm.pipeline_workspace_bytes(W, H, R, H_, B), dtype=torch.uint8, device=dev))

    # C4 with 1 % dropout holes: every tile takes the hole-aware path
    B = 512
    d, lab, K = scenegen.stair_stream(0, B, W, H, REGIONS, device=dev)
    for i in range(B):
        d[i] = scenegen.dropout(d[i], 0.01, 1000 + i, i)
    bb = bufs(B, H, W, REGIONS, HYPS)
    ms = _time_pipeline(pm, d, lab, K, ITERS, REGIONS, HYPS, 0, 5, 2, bb)
    st = stage_times(pm, d, lab, K, ITERS, REGIONS, HYPS, 0, bb[3], bb[0], bb[1], bb[2], reps=3)
    # the same frames through the opt-in PM_ADF_ENGINE_HOLES (fix-up walk), ADF stage alone
    hf = lambda: pm.adf_filter(d, K, LAM, KAPPA, ITERS, out=bb[0], normals_out=bb[1], workspace=bb[3],
                               engine=pm.ENGINE_HOLES)
    for _ in range(2):
        hf()
    e0, e1 = _events(2)
    e0.record()
    for _ in range(5):
        hf()
    e1.record()
    torch.cuda.synchronize()
    res["C4_holes_1pct"] = {"value": B / (ms / 1e3), "unit": "frames/s", "frames_per_step": B, "ms_per_step": ms,
                            "stages_ms": st, "adf_normals_ms_engine_holes": e0.elapsed_time(e1) / 5,
                            "workload": "C4 stream with 1 % hash-selected dropout holes per frame (the default "
                                        "AUTO engine, which runs the hole engine while recent calls met invalid "
                                        "pixels; adf_normals_ms_engine_holes: the ADF stage with "
                                        "PM_ADF_ENGINE_HOLES explicitly)"}
    del d, lab, bb
    torch.cuda.empty_cache()

    # C2: one 640x480 frame, N=20, R=32, H=64 -- per-frame latency, eager launches and a CUDA graph
    fr = scenegen.make_config("C2", device=dev)
    d1 = fr["depth"].to(dev)[None].contiguous()
    l1 = fr["labels"].to(dev)[None].contiguous()
    bb = bufs(1, fr["H"], fr["W"], fr["n_regions"], fr["n_hyp"])
    call = lambda: pm.process_frames(d1, l1, fr["K"], LAM, KAPPA, fr["iters"], fr["n_regions"], fr["n_hyp"], TAU,
                                     SEED, depth_out=bb[0], normals_out=bb[1], planes_out=bb[2], workspace=bb[3])
    eager = _time_pipeline(pm, d1, l1, fr["K"], fr["iters"], fr["n_regions"], fr["n_hyp"], 0, 200, 20, bb)
    s = torch.cuda.Stream(device=dev)
    s.wait_stream(torch.cuda.current_stream(dev))
    with torch.cuda.stream(s):
        for _ in range(3):
            call()
    torch.cuda.current_stream(dev).wait_stream(s)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        call()
    ref = bb[2].clone()
    for _ in range(20):
        g.replay()
    torch.cuda.synchronize()
    e0, e1 = _events(2)
    n = 300
    e0.record()
    for _ in range(n):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    graph_ms = e0.elapsed_time(e1) / n
    same = bool(torch.equal(bb[2], ref))
    res["C2_single_frame"] = {
        "latency_ms_eager": eager, "latency_ms_graph": graph_ms, "hz_graph": 1e3 / graph_ms,
        "graph_replay_bitwise_equal": same, "kernels_per_frame": pm.pipeline_kernel_launches(fr["iters"],
                                                                                           fr["n_regions"]),
        "workload": "BASELINE.json configs[1]: one 640x480 D435-noise G-STAIR frame, N=20, R=32, H=64",
        "paper_context": "'>30 Hz' (P:10), 7.5 ms per frame (P:501), 'below 15 ms' (P:539) on the paper's own "
                         "hardware (RTX 4060 laptop class, P:430) -- context, not a target"}
    del d1, l1, bb, g
    torch.cuda.empty_cache()

    # C3 (1280x720 spiral, N=50, R=128 x 256 hypotheses) and C5 (4096x3072 terrain, N=100, R=1024)
    for name, B in (("C3", 32), ("C5", 4)):
        frs = [scenegen.make_config(name, frame=i, device=dev) for i in range(B)]
        fr = frs[0]
        d = torch.stack([f["depth"].to(dev) for f in frs]).contiguous()
        lab = torch.stack([f["labels"].to(dev) for f in frs]).contiguous()
        del frs
        bb = bufs(B, fr["H"], fr["W"], fr["n_regions"], fr["n_hyp"])
        ms = _time_pipeline(pm, d, lab, fr["K"], fr["iters"], fr["n_regions"], fr["n_hyp"], 0, 3, 1, bb)
        st = stage_times(pm, d, lab, fr["K"], fr["iters"], fr["n_regions"], fr["n_hyp"], 0, bb[3], bb[0], bb[1],
                         bb[2], reps=3)
        rf, rr = rooflines(fr["W"], fr["H"], B, fr["iters"], fr["n_hyp"], _labelled(bb[0], lab, fr["n_regions"]),
                           st, clk_mhz, hbm_peak)
        res[name] = {"value": B / (ms / 1e3), "unit": "frames/s", "frames_per_step": B, "ms_per_step": ms,
                     "adf_alu_frac": rf["frac"], "adf_hbm_frac": rf["hbm"]["frac"], "score_issue_frac": rr["frac"],
                     "stages_ms": st,
                     "workload": f"BASELINE.json {name}: {fr['W']}x{fr['H']}, N={fr['iters']}, "
                                 f"R={fr['n_regions']}, H={fr['n_hyp']}"}
        del d, lab, bb
        torch.cuda.empty_cache()
    return res


def run_cuda(args, rank, world, local_rank):
    import torch
    import torch.distributed as dist

    import paper_2411_01919_b200 as pm
    import scenegen

    dev = torch.device("cuda", local_rank)
    torch.cuda.set_device(dev)
    first, B = shard(rank, args.frames_per_rank)
    # inputs: distinct frames of the C4 stream, generated on the device and kept resident in HBM
    depth, labels, K = scenegen.stair_stream(first, B, W, H, REGIONS, device=dev)
    depth_out = torch.empty_like(depth)
    normals = torch.empty(B, 3, H, W, dtype=torch.float32, device=dev)
    planes = torch.empty(B, REGIONS, pm.PLANE_WORDS, dtype=torch.int32, device=dev)
    ws = torch.empty(pm.pipeline_workspace_bytes(W, H, REGIONS, HYPS, B), dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream(dev)

    def step():
        pm.process_frames(depth, labels, K, LAM, KAPPA, ITERS, REGIONS, HYPS, TAU, SEED, first_frame_id=first,
                          depth_out=depth_out, normals_out=normals, planes_out=planes, workspace=ws)

    def barrier():
        if world > 1:
            dist.barrier()

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize(dev)
    barrier()
    torch.cuda.synchronize(dev)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    old_switch = sys.getswitchinterval()
    sys.setswitchinterval(2e-4)          # let the NVML sampler thread run between launches
    with ClockSampler(dev.index if dev.index is not None else 0) as clocks:
        ev0.record(stream)
        for _ in range(args.steps):
            step()
        ev1.record(stream)
        while not ev1.query():           # poll (GIL released) so the sampler thread keeps sampling
            time.sleep(0.0005)
        torch.cuda.synchronize(dev)
    sys.setswitchinterval(old_switch)
    barrier()
    torch.cuda.synchronize(dev)
    ms = ev0.elapsed_time(ev1)
    t = torch.tensor([ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_max = float(t.item())
    value = world * B * args.steps / (ms_max / 1e3)

    # ---- per-stage / per-kernel times (same launch configuration, same stream), for the rooflines
    st = stage_times(pm, depth, labels, K, ITERS, REGIONS, HYPS, first, ws, depth_out, normals, planes,
                     reps=max(3, min(args.steps, 10)))
    peak, peak_src = _peaks()
    clk = clocks.summary().get("sm_mhz") or clocks.max_mhz or 1965
    roof, rs_roof = rooflines(W, H, B, ITERS, HYPS, _labelled(depth_out, labels, REGIONS), st, clk, peak,
                              _ncu_traffic())
    roof["hbm"]["peak_source"] = peak_src
    roof["clock_mhz"] = clk
    rs_roof["clock_mhz"] = clk
    # ---- e2e: host-resident inputs through the public C-ABI host entry
    # (pm_process_frames_host): pinned sensor-native uint16 depth (mm) and
    # the region labels as row runs (PM_LABELS_RUNS: piecewise-constant label
    # images take a few KB per frame; the paper's regions are polygons)
    # in, plane table out; the H2D of every input byte and the D2H of the
    # plane table inside the timed region, chunked and overlapped with the
    # kernels.  (Frames are mm-quantised by the D435 noise model, so the
    # uint16 form is lossless up to f32 rounding of mm * 1e-3.)  The dense
    # uint8 label image (3 B/px in total) is measured alongside.
    h_mm = torch.round(depth.double() * 1000).clamp(0, 65535).to(torch.int32).to(torch.uint16).cpu().pin_memory()
    lab_cpu = labels.cpu()
    h_lab = torch.where(lab_cpu < 0, torch.full_like(lab_cpu, 0xFF), lab_cpu).to(torch.uint8).pin_memory()
    h_runs = pm.encode_label_runs(lab_cpu).pin_memory()
    h_planes = torch.empty(B, REGIONS, pm.PLANE_WORDS, dtype=torch.int32).pin_memory()
    chunk = args.e2e_chunk
    arena = torch.empty(max(pm.host_pipeline_arena_bytes(W, H, REGIONS, HYPS, chunk, pm.DEPTH_U16_MM, f)
                            for f in (pm.LABELS_U8, pm.LABELS_RUNS)), dtype=torch.uint8, device=dev)
    del ws
    torch.cuda.empty_cache()

    def e2e_run(lab_host, sync=True):
        # sync=False: pm_process_frames_host_async per step (the next step's
        # uploads run under this step's last kernels); the timed region ends
        # with the stream that waits for every step's last download
        def e2e_step():
            pm.process_frames_host(h_mm, lab_host, K, LAM, KAPPA, ITERS, REGIONS, HYPS, TAU, SEED,
                                   first_frame_id=first, chunk_frames=chunk, planes_out=h_planes, arena=arena,
                                   device=dev, sync=sync)
        for _ in range(max(1, args.warmup)):
            e2e_step()
        torch.cuda.synchronize(dev)
        barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(args.steps):
            e2e_step()
        e1.record(stream)
        torch.cuda.synchronize(dev)
        te = torch.tensor([e0.elapsed_time(e1)], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(te, op=dist.ReduceOp.MAX)
        return world * B * args.steps / (float(te.item()) / 1e3)

    e2e_value = e2e_run(h_runs, sync=False)
    e2e_sync = e2e_run(h_runs)
    e2e_dense = e2e_run(h_lab)
    e2e_h2d = B * W * H * 2 + h_runs.nbytes
    e2e_d2h = B * REGIONS * 48
    del arena
    torch.cuda.empty_cache()

    # ---- final gather of the plane tables (the only collective)
    gather_tables(planes, world, rank)

    # ---- the other configs and the per-frame context (rank 0, N = 1)
    extra = None
    if rank == 0 and world == 1 and not args.no_extra:
        extra = extra_configs(pm, dev, clk, peak)

    # ---- oracle baseline on the host cores (rank 0, N = 1 only)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        import oracle
        oracle.build()
        cores = _cpu_cores()
        frames = [(depth[0].cpu().numpy(), labels[0].cpu().numpy())]
        _, t1 = _oracle_throughput(frames, K, first, 1)
        n = int(min(max(cores, round(args.cpu_seconds / max(t1, 1e-3))), 8 * cores, B))
        frames = [(depth[i].cpu().numpy(), labels[i].cpu().numpy()) for i in range(n)]
        fps, wall = _oracle_throughput(frames, K, first, cores)
        cpu = {"value": fps, "unit": "frames/s", "cores": cores, "kind": "oracle",
               "sample": f"{n} frames of the same stream ({wall:.1f} s wall, ~{t1 * n:.0f} s of CPU work; "
                         f"1 frame on 1 core: {t1 * 1e3:.0f} ms)", "cpu_model": _cpu_model()}

    launches_per_step = pm.pipeline_kernel_launches(ITERS, REGIONS)
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "frames/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_max / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": WORKLOAD,
                       "frames_per_rank": B, "global_frames_per_step": world * B,
                       "l2": f"inputs larger than L2 ({B * W * H * 8 / 2**20:.0f} MiB depth+labels per rank)",
                       "parallelism": f"frame-sharded x{world}"},
            "roofline": roof,
            "ransac_roofline": rs_roof,
            "stages_ms": st,
            "configs": extra,
            "cpu_baseline": cpu,
            "e2e": {"value": e2e_value, "unit": "frames/s", "h2d_bytes_per_step": e2e_h2d,
                    "d2h_bytes_per_step": e2e_d2h,
                    "api": "pm_process_frames_host_async per step (uint16 mm depth + row-run labels "
                           f"PM_LABELS_RUNS, pinned; {chunk}-frame chunks, copies overlapped with the kernels and "
                           "with the previous step)",
                    "synchronous_calls": {"value": e2e_sync},
                    "dense_uint8_labels": {"value": e2e_dense, "h2d_bytes_per_step": B * W * H * 3}},
            "gpu_launches": launches_per_step * args.steps,
            "clocks": clocks.summary(),
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
    return 0


def _free_port():
    import socket
    with socket.socket(socket.AF_INET, socket.SOCK_STREAM) as so:
        so.bind(("127.0.0.1", 0))
        return so.getsockname()[1]


def _self_launch(n):
    """`bench.py --gpus N` outside torchrun: start N ranks (one per GPU, NCCL)
    through torch.distributed.run on this node, exactly as the driver does."""
    import torch
    have = torch.cuda.device_count()
    if have < n:
        print(json.dumps({"error": f"--gpus {n} needs {n} visible GPUs, found {have}"}), flush=True)
        return 2
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")            # NCCL's communicator log (nranks) on stderr
    env.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    env.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", f"--master-port={_free_port()}", os.path.abspath(__file__)] + sys.argv[1:]
    import subprocess
    return subprocess.call(cmd, env=env)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="cuda", choices=["cuda", "reference"])
    ap.add_argument("--frames-per-rank", type=int, default=512)
    ap.add_argument("--cpu-seconds", type=float, default=15.0, help="CPU work budget of the oracle baseline")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-extra", action="store_true", help="skip the C2/C3/C5/holes extra configs")
    ap.add_argument("--e2e-chunk", type=int, default=256, help="frames per chunk of the host pipeline")
    args = ap.parse_args()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        return run_reference(args, rank, world)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return _self_launch(args.gpus)
    if world > 1:
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local_rank)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    try:
        return run_cuda(args, rank, world, local_rank)
    finally:
        if world > 1:
            import torch.distributed as dist
            dist.destroy_process_group()


if __name__ == "__main__":
    sys.exit(main())
