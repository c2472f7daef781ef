"""H2D bandwidth with one, two and four concurrent copy streams (12 MiB chunks
round-robin over the streams), pinned host memory -> HBM."""
import time

import torch

n = 4 << 30
h = torch.empty(n, dtype=torch.uint8, pin_memory=True)
h.fill_(1)
d = torch.empty(n, dtype=torch.uint8, device="cuda")
chunk = 12 << 20
for ns in (1, 2, 4, 1, 2):
    ss = [torch.cuda.Stream() for _ in range(ns)]
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for i, o in enumerate(range(0, n, chunk)):
        with torch.cuda.stream(ss[i % ns]):
            d[o:o + chunk].copy_(h[o:o + chunk], non_blocking=True)
    torch.cuda.synchronize()
    print(f"{ns} streams: {n / (time.perf_counter() - t0) / 1e9:.1f} GB/s", flush=True)
