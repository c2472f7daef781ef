"""Streamed-upload probe: public selected_inverse on a host matrix, repeated,
before and after a device-resident run (TIB_HOST_TIMING=1 phase marks)."""
import os
import sys
import time

sys.path.insert(0, ".")
os.environ["TIB_HOST_TIMING"] = "1"
import paper_2504_19171_b200 as tib  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "large"
n, w, t, b = {"large": (200000, 2000, 200, 512), "medium": (100000, 1000, 100, 256)}[cfg]
m = tib.generate(n, w, t, 1.0, seed=42, tile_size=b)


def call(tag):
    t0 = time.perf_counter()
    r = tib.selected_inverse(m, "pattern")
    r.diagonal()
    print(f"{tag}: {1e3 * (time.perf_counter() - t0):.1f} ms", file=sys.stderr, flush=True)
    del r


for k in range(4):
    call(f"cold-process rep {k}")
print(tib.bench_resident(m, 3, 1), file=sys.stderr, flush=True)
for k in range(3):
    call(f"after-resident rep {k}")
