#!/bin/bash
# Round profile set (run under gpurun from the repo root), outputs in gpurun_out/:
#   bench_$1.json       the default bench line (no ncu)
#   launches_$1.csv     per-launch gpu__time_duration + DRAM bytes, 2 steps of the bench workload (512 frames)
#   full_$1.ncu-rep     --set full of one ADF pass (plain + fused) and the RANSAC kernels, 64 frames
set -e
mkdir -p gpurun_out
timeout 600 python bench.py > gpurun_out/bench_$1.json 2> gpurun_out/bench_$1.err
P="python tools/profile_step.py --frames 512 --reps 2"
timeout 300 $P > gpurun_out/plain_$1.log 2>&1
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
  -k "regex:adf_|compact_|ransac_" --csv --log-file gpurun_out/launches_$1.csv $P > gpurun_out/ncu_l_$1.log 2>&1
Q="python tools/profile_step.py --frames 64 --reps 1"
timeout 300 $Q > gpurun_out/plain2_$1.log 2>&1
timeout 1200 ncu --set full --import-source on --clock-control none \
  -k "regex:adf_pass|compact_count|compact_scatter|ransac_score|ransac_refit|ransac_hyp" -c 10 \
  -o gpurun_out/full_$1 $Q > gpurun_out/ncu_f_$1.log 2>&1
