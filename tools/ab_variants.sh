#!/bin/bash
# A/B of prebuilt libpmap_<name>.so variants against the default build on one
# box: tools/ab_variants.sh <name>... ; the parity tests matching -k $AB_TESTS
# (default "ransac") per variant,
# then two bench rounds per variant (value, stage times).
B='python bench.py --no-cpu-baseline --steps 20 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d[\"value\"]), d[\"stages_ms\"])"'
for v in "$@"; do PMAP_LIB_VARIANT=$v timeout 200 python -m pytest tests -m gpu -q -k "${AB_TESTS:-ransac}" 2>&1 | tail -1 | sed "s/^/$v tests: /"; done
for i in 1 2; do for v in "" "$@"; do echo "== ${v:-default}"; PMAP_LIB_VARIANT=$v timeout 300 bash -c "$B"; done; done
