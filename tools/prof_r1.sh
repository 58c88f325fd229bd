#!/bin/bash
# ncu capture used for profiles/ (run under gpurun from the repo root)
set -e
mkdir -p gpurun_out
K='regex:adf_|compact_|ransac_'
P="python tools/profile_step.py --frames 512 --reps 2"
timeout 300 $P > gpurun_out/plain.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k "$K" --csv --log-file gpurun_out/launches_r1.csv $P > gpurun_out/ncu1.log 2>&1
Q="python tools/profile_step.py --frames 64 --reps 1"
timeout 300 $Q > gpurun_out/plain2.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k "$K" -c 12 -o gpurun_out/prof_r1 $Q > gpurun_out/ncu2.log 2>&1
