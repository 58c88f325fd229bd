#!/bin/bash
# A/B of the score kernel's counting split (PM_SCORE_FADD_MASK in csrc/ransac.cu):
# build libpmap_M<mask>.so for masks 0 1 7 15 beforehand (set the #define,
# make, copy), run on one box with the default build as a fifth arm; checks
# the count-exactness tests per variant, then two bench rounds per variant.
B='python bench.py --no-cpu-baseline --steps 20 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d[\"value\"]), d[\"stages_ms\"])"'
for v in M0 M1 M7 M15; do PMAP_LIB_VARIANT=$v timeout 200 python -m pytest tests -m gpu -q -k "ransac_counts_default or ransac_bit_exact" 2>&1 | tail -1 | sed "s/^/$v tests: /"; done
for i in 1 2; do for v in "" M0 M1 M7 M15; do echo "== ${v:-M5}"; PMAP_LIB_VARIANT=$v bash -c "$B"; done; done
