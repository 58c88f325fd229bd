#!/bin/bash
# DRAM traffic + duration per launch of every pmap kernel on the bench workload (512 frames)
set -e
mkdir -p gpurun_out
P="python tools/profile_step.py --frames 512 --reps 2"
timeout 300 $P > gpurun_out/plain_tr.log 2>&1
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
  -k "regex:adf_|compact_|ransac_" --csv --log-file gpurun_out/$1.csv $P > gpurun_out/ncu_tr.log 2>&1
