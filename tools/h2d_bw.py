"""Raw pinned host->device copy bandwidth on this box (the e2e ceiling)."""
import time

import torch

dev = torch.device("cuda", 0)
for mb in (64, 256, 1024):
    n = mb << 20
    h = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    d = torch.empty(n, dtype=torch.uint8, device=dev)
    s = torch.cuda.Stream()
    for _ in range(3):
        with torch.cuda.stream(s):
            d.copy_(h, non_blocking=True)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(s):
        e0.record()
        for _ in range(10):
            d.copy_(h, non_blocking=True)
        e1.record()
    torch.cuda.synchronize()
    print(f"H2D {mb} MiB: {10 * n / (e0.elapsed_time(e1) / 1e3) / 1e9:.1f} GB/s")
    with torch.cuda.stream(s):
        e0.record()
        for _ in range(10):
            h.copy_(d, non_blocking=True)
        e1.record()
    torch.cuda.synchronize()
    print(f"D2H {mb} MiB: {10 * n / (e0.elapsed_time(e1) / 1e3) / 1e9:.1f} GB/s")
