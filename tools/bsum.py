"""One-line summaries of bench JSON lines (files given on the command line)."""
import json
import sys

for f in sys.argv[1:]:
    for line in open(f):
        if line.startswith("{"):
            d = json.loads(line)
            g = d.get("e2e_device_generated") or {}
            print(f"{f}: value {d['value']:.2f} step {d['ms_per_step']:.1f} ms (factor {d['ms_factorize_sweep']:.1f}, "
                  f"phase2 {d['ms_phase2_sweep']:.1f}) e2e {d['e2e']['value']:.2f} ({1e3 * d['e2e']['seconds_per_matrix']:.1f} ms/matrix)"
                  f" gen {g.get('value', float('nan')):.2f} frac {d['roofline']['frac']:.3f}")
