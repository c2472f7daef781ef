"""Public selected_inverse calls on a device-generated large matrix (for an
ncu launch list of the generator / permutation kernels next to the sweeps)."""
import sys
import time

sys.path.insert(0, ".")
import paper_2504_19171_b200 as tib  # noqa: E402

m = tib.generate(200000, 2000, 200, 1.0, seed=42, tile_size=512, device=0)
for rep in range(int(sys.argv[1]) if len(sys.argv) > 1 else 1):
    t0 = time.perf_counter()
    r = tib.selected_inverse(m, "pattern", device=0)
    r.diagonal()
    print(f"rep {rep}: {1e3 * (time.perf_counter() - t0):.1f} ms", flush=True)
    del r
