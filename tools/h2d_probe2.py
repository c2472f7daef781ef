"""H2D chunked copies with a 4-byte counter write after each chunk: as a tiny
H2D memcpy, or as a stream memory operation (cuStreamWriteValue32)."""
import ctypes
import time

import torch

n = 4 << 30
h = torch.empty(n, dtype=torch.uint8, pin_memory=True)
h.fill_(1)
d = torch.empty(n, dtype=torch.uint8, device="cuda")
one = torch.ones(1, dtype=torch.int32).pin_memory()
ctr = torch.zeros(4096, dtype=torch.int32, device="cuda")
s = torch.cuda.Stream()
cu = ctypes.CDLL("libcuda.so.1")
cu.cuStreamWriteValue32.argtypes = [ctypes.c_void_p, ctypes.c_uint64, ctypes.c_uint32, ctypes.c_uint]
for chunk in (12 << 20, 6 << 20):
    for mode in ("none", "memcpy", "writevalue"):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        with torch.cuda.stream(s):
            for i, o in enumerate(range(0, n, chunk)):
                d[o:o + chunk].copy_(h[o:o + chunk], non_blocking=True)
                if mode == "memcpy":
                    ctr[i:i + 1].copy_(one, non_blocking=True)
                elif mode == "writevalue":
                    r = cu.cuStreamWriteValue32(ctypes.c_void_p(s.cuda_stream), ctypes.c_uint64(ctr.data_ptr() + 4 * i), 1, 0)
                    assert r == 0, r
        s.synchronize()
        dt = time.perf_counter() - t0
        print(f"chunk {chunk >> 20} MiB, counter {mode}: {n / dt / 1e9:.1f} GB/s", flush=True)
