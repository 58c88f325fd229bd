#!/bin/bash
# Per-pass ADF kernel durations and occupancy limits for libpmap_A.so vs the
# current libpmap.so (ncu launch lists; compare the two, not absolutes).
mkdir -p gpurun_out
M=gpu__time_duration.sum,launch__occupancy_limit_shared_mem,launch__occupancy_limit_registers,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__inst_executed.sum
for v in A B; do
  if [ $v = A ]; then export PMAP_LIB_VARIANT=A; else unset PMAP_LIB_VARIANT; fi
  ncu --metrics $M --clock-control none -k regex:adf_pass --csv --log-file gpurun_out/adf_passes_$v.csv \
      python tools/sweep_adf_div.py > gpurun_out/adf_passes_$v.log 2>&1
done
