"""Host-side phase timing of the public calls (TIB_HOST_TIMING=1), run under gpurun."""
import os
import sys
import time

sys.path.insert(0, ".")
os.environ["TIB_HOST_TIMING"] = "1"
import paper_2504_19171_b200 as tib  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "batch"
if cfg == "batch":
    for dev in (False, True):
        ms = [tib.generate(50000, 500, 50, 1.0, seed=1000 + k, tile_size=128, device=0 if dev else None)
              for k in range(64)]
        for rep in range(2):
            t0 = time.perf_counter()
            tib.selected_inverse_batch(ms)
            print(f"batch device_gen={dev} rep {rep}: {1e3 * (time.perf_counter() - t0):.1f} ms", file=sys.stderr,
                  flush=True)
elif cfg == "kronecker":
    m = tib.generate_kronecker(tile_size=512, **tib.KRONECKER_CONFIG)
    for rep in range(2):
        t0 = time.perf_counter()
        r = tib.selected_inverse(m, "pattern")
        r.diagonal()
        print(f"kronecker rep {rep}: {1e3 * (time.perf_counter() - t0):.1f} ms", file=sys.stderr, flush=True)
else:
    for dev in (False, True):
        m = tib.generate(200000, 2000, 200, 1.0, seed=42, tile_size=512, device=0 if dev else None)
        for rep in range(2):
            t0 = time.perf_counter()
            r = tib.selected_inverse(m, "pattern")
            r.diagonal()
            print(f"large device_gen={dev} rep {rep}: {1e3 * (time.perf_counter() - t0):.1f} ms", file=sys.stderr,
                  flush=True)
