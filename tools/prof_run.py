"""Profiling driver: one fused factorize + selected inversion at a named config
(run under ncu; never a bench number)."""
import sys

sys.path.insert(0, ".")
import paper_2504_19171_b200 as tib  # noqa: E402

CONFIGS = {
    "small": (10000, 200, 50, 128),
    "medium": (100000, 1000, 100, 256),
    "large": (200000, 2000, 200, 512),
    "mini": (20000, 2000, 200, 512),
}

if __name__ == "__main__":
    n, w, t, b = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "small"]
    reps = int(sys.argv[2]) if len(sys.argv) > 2 else 1
    m = tib.generate(n, w, t, 1.0, seed=42, tile_size=b)
    print(tib.bench_resident(m, reps, 0))
