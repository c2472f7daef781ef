"""Summarise a dataflow task trace written with TIB_TRACE=<prefix> (engine.cpp
write_trace): per queue busy / waiting time, per task-kind durations."""
import sys

import numpy as np


def load(path):
    with open(path, "rb") as f:
        hdr = np.frombuffer(f.read(32), np.int64)
        ntask, batch, nq0, nb = (int(x) for x in hdr)
        kinds = np.frombuffer(f.read(ntask), np.uint8)
        segc = np.frombuffer(f.read(4 * ntask), np.int32)
        rec = np.frombuffer(f.read(), np.uint64).reshape(-1, 4)
    return ntask, batch, nq0, nb, kinds, segc, rec


def report(path):
    ntask, batch, nq0, nb, kinds, segc, rec = load(path)
    ok = rec[:, 2] > 0
    rec = rec[ok]
    claim, ready, done = (rec[:, i].astype(np.float64) for i in range(3))
    task = (rec[:, 3] >> 32).astype(np.int64)
    sm = (rec[:, 3] & 0xFFFF).astype(np.int64)
    t0 = claim.min()
    span = (done.max() - t0) / 1e3
    q0 = task < nq0
    print(f"{path}: tasks={len(rec)} (q0 {q0.sum()}, q1 {(~q0).sum()}) span={span:.1f} us")
    for name, m in (("q0/crit", q0), ("q1/bulk", ~q0)):
        if m.sum() == 0:
            continue
        wait = (ready[m] - claim[m]).sum() / 1e3
        busy = (done[m] - ready[m]).sum() / 1e3
        workers = len(np.unique(sm[m]))
        print(f"  {name}: busy {busy:.0f} us, waiting {wait:.0f} us (wait share {wait / (wait + busy):.2f}), "
              f"SMs {workers}, first {(claim[m].min() - t0) / 1e3:.1f} last-done {(done[m].max() - t0) / 1e3:.1f} us")
    dur = (done - ready) / 1e3
    k = kinds[task]
    s = segc[task]
    print("  leaf tasks: n=%d mean %.1f us  p50 %.1f  max %.1f" % ((k == 1).sum(), dur[k == 1].mean() if (k == 1).any() else 0,
          np.median(dur[k == 1]) if (k == 1).any() else 0, dur[k == 1].max() if (k == 1).any() else 0))
    for sc in sorted(set(s[(k == 0)].tolist())):
        m = (k == 0) & (s == sc)
        for name, qm in (("q0", q0), ("q1", ~q0)):
            mm = m & qm
            if mm.sum():
                print(f"  gemm seg_count={sc} {name}: n={mm.sum()} mean {dur[mm].mean():.1f} us p50 {np.median(dur[mm]):.1f}")
    # utilisation timeline (10 buckets)
    edges = np.linspace(t0, done.max(), 11)
    busy_t = []
    for a, b in zip(edges[:-1], edges[1:]):
        ov = np.clip(np.minimum(done, b) - np.maximum(ready, a), 0, None).sum()
        busy_t.append(ov / ((b - a) * 2 * len(np.unique(sm))) if b > a else 0)
    print("  busy fraction per tenth of the sweep:", " ".join(f"{x:.2f}" for x in busy_t))


if __name__ == "__main__":
    for p in sys.argv[1:]:
        report(p)
