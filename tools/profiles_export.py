#!/usr/bin/env python
"""Export the round's ncu evidence into profiles/ (tracked):
  python tools/profiles_export.py <tag> <round-label>
reads gpurun_out/launches_<tag>.csv (launch list: time + DRAM bytes, 2 steps
of the bench workload, 512 frames) and gpurun_out/full_<tag>.ncu-rep (--set
full, 64 frames) and writes
  profiles/<round>_launches_512frames.csv   the raw launch list
  profiles/<round>_ncu_full_summary.csv     one row per captured kernel: key metrics
  profiles/adf_traffic.json                 the ADF stage's DRAM bytes (bench.py roofline.traffic)"""
import csv
import json
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
tag, rnd = sys.argv[1], sys.argv[2]
out = os.path.join(ROOT, "profiles")
lc = os.path.join(ROOT, "gpurun_out", f"launches_{tag}.csv")
shutil.copy(lc, os.path.join(out, f"{rnd}_launches_512frames.csv"))

# ---- ADF stage traffic from the launch list (first step's 5 adf passes)
lines = open(lc).read().splitlines()
start = [i for i, l in enumerate(lines) if l.startswith('"ID"')][0]
rows = list(csv.reader(lines[start:]))
hdr = rows[0]
ii, ki, mi, vi, ui = (hdr.index(k) for k in ("ID", "Kernel Name", "Metric Name", "Metric Value", "Metric Unit"))
mult = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1.0, "usecond": 1e3, "msecond": 1e6}
launch = {}
order = []
for r in rows[1:]:
    key = int(r[ii])
    if key not in launch:
        launch[key] = {"kernel": r[ki].split("(")[0].replace("void ", "").split("::")[-1]}
        order.append(key)
    launch[key][r[mi]] = float(r[vi].replace(",", "")) * mult.get(r[ui], 1.0)
adf = [launch[k] for k in order if "adf_pass" in launch[k]["kernel"]][:5]
stage = sum(l["dram__bytes_read.sum"] + l["dram__bytes_write.sum"] for l in adf)
json.dump({
    "source": f"ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum "
              f"(tools/prof_round.sh), 512 C4 frames, {rnd}",
    "kernel": "adf_pass_kernel, one ADF+normals stage = 5 launches (4 x T=4 sweeps + 1 fused T=4 + normals)",
    "bytes_per_launch": stage / len(adf),
    "bytes_per_stage": stage,
    "alg_bytes_per_stage": 20 * 640 * 480 * 512,
    "launches": [{"kernel": l["kernel"], "dram_read": l["dram__bytes_read.sum"],
                  "dram_write": l["dram__bytes_write.sum"], "ns": l["gpu__time_duration.sum"]} for l in adf],
    "ncu_stage_ns": sum(l["gpu__time_duration.sum"] for l in adf),
}, open(os.path.join(out, "adf_traffic.json"), "w"), indent=1)

# ---- --set full summary
rep = os.path.join(ROOT, "gpurun_out", f"full_{tag}.ncu-rep")
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rr = list(csv.reader(raw.splitlines()))
H = rr[0]
U = dict(zip(rr[0], rr[1]))     # units row
keys = [("duration_us", "gpu__time_duration.sum"), ("issue_active_pct", "sm__inst_issued.avg.pct_of_peak_sustained_active"),
        ("warp_instr", "smsp__inst_executed.sum"), ("occupancy_pct", "sm__warps_active.avg.pct_of_peak_sustained_active"),
        ("regs", "launch__registers_per_thread"), ("dram_read", "dram__bytes_read.sum"),
        ("dram_write", "dram__bytes_write.sum"), ("dram_pct", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"),
        ("fma_pipe_pct", "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active"),
        ("alu_pipe_pct", "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active"),
        ("xu_pipe_pct", "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active"),
        ("smem_wavefronts_pct", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed")]
with open(os.path.join(out, f"{rnd}_ncu_full_summary.csv"), "w", newline="") as fh:
    w = csv.writer(fh)
    w.writerow(["kernel"] + [f"{k} [{U.get(m, '')}]" for k, m in keys] + ["top_stalls_per_issue"])
    for r in rr[2:]:
        d = dict(zip(H, r))
        st = []
        for h, v in d.items():
            if h.startswith("smsp__average_warps_issue_stalled") and h.endswith("_per_issue_active.ratio"):
                try:
                    st.append((float(v), h[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]))
                except ValueError:
                    pass
        st = "; ".join(f"{n} {v:.2f}" for v, n in sorted(st, reverse=True)[:6])
        w.writerow([d["Kernel Name"].split("(")[0].replace("void ", "").split("::")[-1]] + [d.get(m, "") for _, m in keys] + [st])
print("exported", tag, "->", rnd)
