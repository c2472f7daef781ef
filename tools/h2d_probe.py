"""H2D bandwidth probe (pinned host memory -> HBM), whole buffer and chunked."""
import time

import torch

n = 4 << 30
h = torch.empty(n, dtype=torch.uint8, pin_memory=True)
h.fill_(1)
d = torch.empty(n, dtype=torch.uint8, device="cuda")
s = torch.cuda.Stream()
for chunk in (n, 256 << 20, 32 << 20, 6 << 20, 2 << 20):
    for rep in range(2):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        with torch.cuda.stream(s):
            for o in range(0, n, chunk):
                d[o:o + chunk].copy_(h[o:o + chunk], non_blocking=True)
        s.synchronize()
        dt = time.perf_counter() - t0
    print(f"chunk {chunk >> 20} MiB: {n / dt / 1e9:.1f} GB/s", flush=True)
# D2H
torch.cuda.synchronize()
t0 = time.perf_counter()
h.copy_(d, non_blocking=True)
torch.cuda.synchronize()
print(f"D2H whole: {n / (time.perf_counter() - t0) / 1e9:.1f} GB/s")

# H2D while the SMs run FP64 GEMMs on another stream
a = torch.randn(8192, 8192, dtype=torch.float64, device="cuda")
c = torch.empty_like(a)
busy = torch.cuda.Stream()
for chunk in (n, 6 << 20):
    torch.cuda.synchronize()
    with torch.cuda.stream(busy):
        for _ in range(40):
            torch.matmul(a, a, out=c)
    t0 = time.perf_counter()
    with torch.cuda.stream(s):
        for o in range(0, n, chunk):
            d[o:o + chunk].copy_(h[o:o + chunk], non_blocking=True)
    s.synchronize()
    dt = time.perf_counter() - t0
    print(f"H2D under DGEMM load, chunk {chunk >> 20} MiB: {n / dt / 1e9:.1f} GB/s", flush=True)
    torch.cuda.synchronize()
