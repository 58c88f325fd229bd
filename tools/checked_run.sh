#!/bin/bash
# Checked build (compute-sanitizer is closed on this pool): the library built
# with -DPM_CHECKED (device bounds checks on the hot kernels' shared- and
# global-memory indices; a failed check traps) runs the sanitize workload,
# the bench workload with and without dropout, and the GPU test suite.
#   bash tools/build_variant.sh checked -DPM_CHECKED   (here, then under gpurun:)
#   bash tools/checked_run.sh > gpurun_out/checked_run.txt 2>&1
export PMAP_LIB_VARIANT=checked
python -c "import paper_2411_01919_b200 as pm; print('library:', pm._lib._name)"
echo "== tools/sanitize_run.py"; timeout 600 python tools/sanitize_run.py; echo "rc $?"
echo "== bench workload (512 C4 frames, hole-free and 1 % dropout, default and HOLES engines)"
timeout 600 python - <<'PY'
import torch, scenegen, paper_2411_01919_b200 as pm
d, lab, K = scenegen.stair_stream(0, 512, 640, 480, 64, device="cuda")
for holes in (0.0, 0.01):
    x = d.clone()
    if holes:
        for i in range(512):
            x[i] = scenegen.dropout(x[i], holes, 1000 + i, i)
    out, nrm, planes = pm.process_frames(x, lab, K, 0.15, 0.03, 20, 64, 64, 0.01, 0x1919)
    for eng in (pm.ENGINE_TILED, pm.ENGINE_HOLES, pm.ENGINE_REG):
        o2, n2 = pm.adf_filter(x, K, 0.15, 0.03, 20, engine=eng)
        assert torch.equal(o2, out)
    torch.cuda.synchronize()
    print("holes", holes, "ok")
PY
echo "rc $?"
echo "== pytest -m gpu"; timeout 1200 python -m pytest tests -q -m gpu 2>&1 | tail -3
