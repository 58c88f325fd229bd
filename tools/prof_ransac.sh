#!/bin/bash
# ncu capture of the RANSAC kernels (64 frames) -> gpurun_out/$1.ncu-rep
set -e
mkdir -p gpurun_out
Q="python tools/profile_step.py --frames 64 --reps 1"
timeout 300 $Q > gpurun_out/plain_rs.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k "regex:ransac_score|ransac_refit|compact_count|compact_scatter" -c 4 -o gpurun_out/$1 $Q > gpurun_out/ncu_rs.log 2>&1
