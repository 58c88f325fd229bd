#!/bin/bash
# Source-level counters (SASS) of one plain ADF pass (the second launch) for
# libpmap_A.so and the current libpmap.so: gpurun_out/adf_src_{A,B}.csv.
mkdir -p gpurun_out
for v in A B; do
  if [ $v = A ]; then export PMAP_LIB_VARIANT=A; else unset PMAP_LIB_VARIANT; fi
  ncu --section SourceCounters --section WarpStateStats --import-source on --clock-control none \
      -k regex:adf_pass_kernel --launch-skip 1 --launch-count 1 -o gpurun_out/adf_src_$v -f \
      python tools/sweep_adf_div.py > gpurun_out/adf_src_$v.log 2>&1
  ncu -i gpurun_out/adf_src_$v.ncu-rep --page source --csv --print-source sass > gpurun_out/adf_src_$v.csv
done
