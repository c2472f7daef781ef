"""Phase timing of the partitioned path with every part in one process
(P parts on one GPU, sequential): per-part phase A / D, the reduced solve;
the parallel time of P GPUs is max(A) + all-reduce + C + max(D)."""
import sys
import time

sys.path.insert(0, ".")
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2504_19171_b200 as tib  # noqa: E402
from paper_2504_19171_b200 import partition as P  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "large"
parts = int(sys.argv[2]) if len(sys.argv) > 2 else 2
n, w, t, b = {"large": (200000, 2000, 200, 512), "medium": (100000, 1000, 100, 256)}[cfg]
m = tib.generate(n, w, t, 1.0, seed=42, tile_size=b)
t0 = time.perf_counter()
ti, tj, pay = m.tiles()
A = P.TileMap(n, b, ti, tj, pay)
bw, na = P.band_of(ti, tj, A.N)
part = P.BandArrowPartition(A.N, bw, parts, na)
print(f"tiles() + map {time.perf_counter() - t0:.2f} s; interiors {[len(x) for x in part.interiors]}", flush=True)
eng = P.DeviceEngine(0)


def tick():
    torch.cuda.synchronize()
    return time.perf_counter()


for rep in range(2):
    rows_last = A.rows(part.last)
    nR = (len(part.reduced) - 1) * b + rows_last
    G = np.zeros((nR, nR))
    ta, state, ld = [], {}, 0.0
    for p in range(parts):
        s0 = tick()
        f, C, _, ldi = P.phase_a(A, part, p, eng)
        P.scatter_reduced(part, p, C, b, rows_last, G)
        ta.append(tick() - s0)
        state[p] = f
        ld += ldi
    s0 = tick()
    S = P.reduced_matrix(A, part, G)
    S = 0.5 * (S + S.T)
    sig_R, ld_S = eng.reduced_inverse(S, b)
    red = P.ReducedResult(sig_R, ld_S, part.reduced)
    tc = tick() - s0
    td = []
    for p in range(parts):
        s0 = tick()
        P.phase_d(A, part, p, state[p], red, eng)
        td.append(tick() - s0)
    print(f"rep {rep}: A {['%.3f' % x for x in ta]} C {tc:.3f} D {['%.3f' % x for x in td]} "
          f"-> parallel estimate {max(ta) + tc + max(td):.3f} s; logdet {ld + ld_S:.6f}", flush=True)
    res = tib.selected_inverse(m, "pattern")
    print(f"single-GPU logdet {res.logdet():.6f}", flush=True)
