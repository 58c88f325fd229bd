#!/bin/bash
# A/B timing on one box: tools/ab.sh "<command>" runs the command alternately
# with libpmap_A.so (saved baseline: cp paper_2411_01919_b200/libpmap.so
# paper_2411_01919_b200/libpmap_A.so before the change) and the current
# libpmap.so, three times each.
for i in 1 2 3; do
  echo "== A"; PMAP_LIB_VARIANT=A bash -c "$1"
  echo "== B"; bash -c "$1"
done
