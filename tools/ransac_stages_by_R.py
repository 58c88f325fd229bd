import sys, os
sys.path.insert(0, os.getcwd())
import torch, bench, scenegen, paper_2411_01919_b200 as pm
B, W, H, NH = 256, 640, 480, 64
for R in (64, 256, 1024):
    d4, lab4, K = scenegen.stair_stream(0, 4, W, H, R, device="cpu")
    d = d4.repeat(B // 4, 1, 1).contiguous().cuda(); lab = lab4.repeat(B // 4, 1, 1).contiguous().cuda()
    ws = torch.empty(pm.pipeline_workspace_bytes(W, H, R, NH, B), dtype=torch.uint8, device="cuda")
    out = torch.empty_like(d); nrm = torch.empty(B, 3, H, W, device="cuda"); pl = torch.empty(B, R, 12, dtype=torch.int32, device="cuda")
    st = bench.stage_times(pm, d, lab, K, 20, R, NH, 0, ws, out, nrm, pl, reps=3)
    print(R, {k: round(v / B * 1e3, 2) for k, v in st.items()}, "us/frame")
