"""A/B of environment knobs read at plan build time: each setting of
`KEY=V[,KEY=V]` runs one config (device resident, 3 timed reps after 2) in its
own process; settings are interleaved over `--rounds` to expose drift.

    python tools/ab_env.py large TIB_C0_PF_P2=0 TIB_C0_PF_P2=1 --rounds 2
"""
import argparse
import json
import os
import subprocess
import sys

CODE = r'''
import json, sys
sys.path.insert(0, ".")
import paper_2504_19171_b200 as tib
cfg = sys.argv[1]
if cfg == "batch":
    r = tib.Resident([tib.generate(50000, 500, 50, 1.0, seed=1000 + k, tile_size=128, device=0) for k in range(64)], device=0)
elif cfg == "kronecker":
    r = tib.Resident(tib.generate_kronecker(tile_size=512, **tib.KRONECKER_CONFIG), device=0)
else:
    n, w, t, b = {"large": (200000, 2000, 200, 512), "medium": (100000, 1000, 100, 256)}[cfg]
    r = tib.Resident(tib.generate(n, w, t, 1.0, seed=42, tile_size=b, device=0), device=0)
r.run(2)
tot, f, p = r.run(3)
print(json.dumps({"ms_step": round(tot / 3, 2), "ms_factor": round(f, 2), "ms_phase2": round(p, 2)}))
'''

ap = argparse.ArgumentParser()
ap.add_argument("config")
ap.add_argument("settings", nargs="+")
ap.add_argument("--rounds", type=int, default=1)
args = ap.parse_args()
for rnd in range(args.rounds):
    for spec in args.settings:
        env = dict(os.environ)
        for kv in spec.split(","):
            if kv:
                k, v = kv.split("=")
                env[k] = v
        out = subprocess.run([sys.executable, "-c", CODE, args.config], env=env, capture_output=True, text=True,
                             timeout=900)
        line = out.stdout.strip().splitlines()[-1] if out.stdout.strip() else out.stderr[-300:]
        print(args.config, rnd, spec, line, flush=True)
