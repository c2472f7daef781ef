"""cuBLAS DGEMM peak on the box (burst best-of-10 and ~4 s sustained), for the
FP64 roofline denominator.  Prints JSON lines."""
import json
import time

import torch

n = 8192
a = torch.randn(n, n, dtype=torch.float64, device="cuda")
b = torch.randn(n, n, dtype=torch.float64, device="cuda")
c = torch.empty_like(a)
for _ in range(3):
    torch.matmul(a, b, out=c)
torch.cuda.synchronize()
best = 1e9
for _ in range(10):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    torch.matmul(a, b, out=c)
    e1.record()
    torch.cuda.synchronize()
    best = min(best, e0.elapsed_time(e1))
print(json.dumps({"kind": "cublas_dgemm_8192_burst", "tflops": 2 * n**3 / best / 1e9, "ms": best}))
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
reps = 0
t0 = time.time()
while time.time() - t0 < 4.0:
    torch.matmul(a, b, out=c)
    reps += 1
    if reps % 8 == 0:
        torch.cuda.synchronize()
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1)
print(json.dumps({"kind": "cublas_dgemm_8192_sustained", "tflops": 2 * n**3 * reps / ms / 1e9, "ms": ms}))
