"""Two-chain path diagnostics: each variant in its own process with a short
watchdog; prints ok / the error."""
import os
import subprocess
import sys

CODE = r'''
import sys, os
sys.path.insert(0, ".")
import numpy as np
import paper_2504_19171_b200 as tib
case = sys.argv[1]
if case == "smoke":
    m = tib.generate(700, 90, 12, 1.0, seed=5, tile_size=64)
elif case == "kron_small":
    m = tib.generate_kronecker(3, 20, 10, 5, tile_size=64)
elif case == "mid":
    m = tib.generate(9000, 600, 70, 1.0, seed=31, tile_size=128)
else:
    n, w, t, b = (int(x) for x in case.split(","))
    m = tib.generate(n, w, t, 1.0, seed=5, tile_size=b)
print("split", tib.two_chain_order(m)[1], "N", m.n_tiles, flush=True)
r = tib.selected_inverse(m, "pattern")
print("logdet", r.logdet())
'''
for case in sys.argv[1:]:
    for env in ({"TIB_SPLIT_STREAMED": "1"}, {"TIB_SPLIT_STREAMED": "1", "TIB_SPLIT_AGENTS": "1"}, {"TIB_STREAM_UPLOAD": "0"}, {"TIB_SPLIT": "0"}):
        e = dict(os.environ, TIB_WATCHDOG_S="5", **env)
        out = subprocess.run([sys.executable, "-c", CODE, case], env=e, capture_output=True, text=True, timeout=300)
        tail = (out.stdout.strip().splitlines() or [""])[-1] if out.returncode == 0 else out.stderr.strip().splitlines()[-1]
        head = (out.stdout.strip().splitlines() or [""])[0]
        print(case, env, "rc", out.returncode, head, "|", tail[:200], flush=True)
