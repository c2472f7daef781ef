"""Device-resident timing of BASELINE config 5 (64 x (50000, 500, 50), b=128) for
tuning sweeps (env knobs are read per run): prints (ms total, ms factor, ms phase 2)."""
import sys

sys.path.insert(0, ".")
import paper_2504_19171_b200 as tib  # noqa: E402

if __name__ == "__main__":
    count = int(sys.argv[1]) if len(sys.argv) > 1 else 64
    b = int(sys.argv[2]) if len(sys.argv) > 2 else 128
    ms = [tib.generate(50000, 500, 50, 1.0, seed=1000 + k, tile_size=b) for k in range(count)]
    r = tib.Resident(ms)
    r.run(2)
    tot, f, p = r.run(3)
    print(f"count={count} b={b} ms/step={tot / 3:.1f} factor={f:.1f} phase2={p:.1f}", flush=True)
