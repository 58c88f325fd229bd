import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, numpy as np
import paper_2411_01919_b200 as pm, scenegen
for (W, H) in [(64, 48), (640, 480)]:
    K = scenegen.intrinsics_for(W, H)
    rng = np.random.default_rng(0)
    d = torch.from_numpy((1.5 + 0.01 * rng.standard_normal((H, W))).astype(np.float32)).cuda()
    for it in (1, 2, 3, 5):
        a, na = pm.adf_filter(d, K, 0.15, 0.03, it, engine=pm.ENGINE_TILED)
        b, nb = pm.adf_filter(d, K, 0.15, 0.03, it, engine=pm.ENGINE_STREAM)
        torch.cuda.synchronize()
        diff = (a != b)
        nd = (na != nb).any(0)
        ys, xs = torch.nonzero(diff, as_tuple=True)
        print(W, H, "iters", it, "depth diffs", int(diff.sum()), "normal diffs", int(nd.sum()),
              "rows", sorted(set(ys.tolist()))[:10], "cols", sorted(set(xs.tolist()))[:10])
