"""Factor / phase-2 sweep times of one config against the number of workers
reserved for the critical queue (TIB_CRIT_WORKERS_FACTOR / _P2 are read when a
plan is built, so each setting runs in its own process)."""
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
    ms = [tib.generate(50000, 500, 50, 1.0, seed=1000 + k, tile_size=128, device=0) for k in range(64)]
    r = tib.Resident(ms, device=0)
else:
    n, w, t, b = {"large": (200000, 2000, 200, 512), "medium": (100000, 1000, 100, 256)}[cfg]
    r = tib.Resident(tib.generate(n, w, t, 1.0, seed=42, tile_size=b, device=0), device=0)
r.run(2)
tot, f, p = r.run(3)
print(json.dumps({"ms_step": tot / 3, "ms_factor": f, "ms_phase2": p}))
'''

cfg = sys.argv[1]
for spec in sys.argv[2:]:
    fa, p2 = spec.split(",")
    env = dict(os.environ, TIB_CRIT_WORKERS_FACTOR=fa, TIB_CRIT_WORKERS_P2=p2, TIB_CRIT_BATCH_FACTOR=fa,
               TIB_CRIT_BATCH_P2=p2)
    out = subprocess.run([sys.executable, "-c", CODE, cfg], env=env, capture_output=True, text=True, timeout=600)
    line = out.stdout.strip().splitlines()[-1] if out.stdout.strip() else out.stderr[-300:]
    print(cfg, spec, line, flush=True)
