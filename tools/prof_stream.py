import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench, paper_2411_01919_b200 as pm, scenegen
T = int(sys.argv[1]) if len(sys.argv) > 1 else 4
d, lab, K = scenegen.stair_stream(0, 64, bench.W, bench.H, bench.REGIONS, device="cuda")
pm.adf_filter(d, K, bench.LAM, bench.KAPPA, bench.ITERS, engine=pm.ENGINE_STREAM, iters_per_pass=T)
torch.cuda.synchronize()
print("ok")
