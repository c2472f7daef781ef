"""Quick GPU parity + timing probe (development tool, run under gpurun)."""
import json
import sys
import time

import numpy as np

sys.path.insert(0, ".")
import paper_2504_19171_b200 as tib  # noqa: E402
from oracle import oracle as O  # noqa: E402


def cmp_case(n, w, t, d, seed, b, sel="pattern"):
    m = tib.generate(n, w, t, d, seed=seed, tile_size=b)
    t0 = time.time()
    res = tib.selected_inverse(m, sel)
    t1 = time.time()
    ref = O.selected_inverse_generated(n, w, t, d, seed, b, sel)
    ti, tj, pay = res.tiles()
    same = list(zip(ti.tolist(), tj.tolist())) == ref["tiles"]
    err = float(np.abs(pay - ref["payload"]).max() / np.abs(ref["payload"]).max())
    out = {"case": [n, w, t, d, seed, b, sel], "pattern_same": same, "sigma_err": err, "gpu_s": t1 - t0}
    if ref["diag"] is not None:
        dg = res.diagonal()
        out["diag_err"] = float(np.max(np.abs(dg - ref["diag"]) / np.abs(ref["diag"])))
    out["logdet_err"] = abs(res.logdet() - ref["logdet"]) / abs(ref["logdet"])
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    a = np.array([[4.0, 2.0], [2.0, 5.0]])
    r = tib.selected_inverse(tib.from_dense(a), "all")
    print("2x2", r.entries(), flush=True)
    for case in [(24, 5, 2, 0.8, 7, 4, "all"), (60, 9, 3, 0.6, 11, 8, "pattern"), (300, 40, 7, 1.0, 3, 32, "all"),
                 (700, 90, 12, 1.0, 5, 64, "pattern"), (1500, 300, 30, 1.0, 9, 128, "pattern"),
                 (2000, 150, 12, 0.2, 4, 256, "pattern"), (3000, 700, 50, 1.0, 1, 512, "pattern"),
                 (10000, 200, 50, 1.0, 42, 128, "pattern")]:
        cmp_case(*case)
    try:
        tib.factorize(tib.from_dense(np.array([[1.0, 2.0], [2.0, 1.0]])))
        print("NOT SPD NOT RAISED")
    except tib.NotSpdError as e:
        print("notspd", e, e.pivot, e.tile_i, e.tile_j)
    for (n, w, t, b) in [(10000, 200, 50, 128), (100000, 1000, 100, 256), (200000, 2000, 200, 512)]:
        t0 = time.time()
        m = tib.generate(n, w, t, 1.0, seed=42, tile_size=b)
        tg = time.time() - t0
        f = sum(tib.task_flops(m))
        ms, mf, mp, ld = tib.bench_resident(m, 3, 1)
        print(json.dumps({"n": n, "b": b, "gen_s": tg, "ms": ms, "ms_factor": mf, "ms_phase2": mp,
                          "tflops": f / ms / 1e9, "logdet": ld}), flush=True)
