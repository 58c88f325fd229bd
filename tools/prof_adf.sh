#!/bin/bash
# ncu capture of the two adf passes (64 frames) -> gpurun_out/$1.ncu-rep
set -e
mkdir -p gpurun_out
Q="python tools/profile_step.py --frames 64 --reps 1"
timeout 300 $Q > gpurun_out/plain_adf.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:adf_pass -c 2 -o gpurun_out/$1 $Q > gpurun_out/ncu_adf.log 2>&1
