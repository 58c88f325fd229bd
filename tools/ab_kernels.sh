#!/bin/bash
# Per-kernel A/B: ncu launch list (gpu__time_duration) of 2 pipeline steps on
# 512 frames for libpmap_A.so and the current libpmap.so, summarised by
# tools/launches.py.  Run under gpurun after tools/ab.sh.
for v in A B; do
  if [ $v = A ]; then export PMAP_LIB_VARIANT=A; else unset PMAP_LIB_VARIANT; fi
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k "regex:adf_|compact_|ransac_" --csv \
    --log-file gpurun_out/abk_$v.csv python tools/profile_step.py --frames 512 --reps 2 > /dev/null 2>&1
  echo "== $v"; python tools/launches.py gpurun_out/abk_$v.csv
done
