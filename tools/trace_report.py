"""Summarise a dataflow task trace written with TIB_TRACE=<prefix> (engine.cpp
write_trace): per-queue busy / waiting time, per task-class durations, and the
critical path -- walked back from the last task through the dependency whose
counter was satisfied last (or, when the task was claimed after its inputs were
ready, through the task that freed its CTA) -- broken down by task class."""
import collections
import sys

import numpy as np

DTASK = np.dtype({
    "names": ["c_off", "c0_off", "cm_off", "diag_off", "p_off", "ldc", "ldc0", "m0", "n0", "seg_begin", "seg_count",
              "dep_begin", "sig_begin", "aux0", "aux1", "poll", "dep_count", "sig_count", "kind", "mode", "c_store",
              "c0_store", "cm_store", "diag_store", "dep2_count", "sig2_count"],
    "formats": ["<i8"] * 5 + ["<i4"] * 11 + ["<u2"] * 2 + ["u1"] * 8,
    "offsets": [0, 8, 16, 24, 32, 40, 44, 48, 52, 56, 60, 64, 68, 72, 76, 80, 88, 90, 92, 93, 94, 95, 96, 97, 98, 99],
    "itemsize": 104,
})
DEP = np.dtype([("counter", "<i4"), ("value", "<i4")])
SEG = np.dtype({
    "names": ["a_off", "b_off", "lda", "ldb", "k_lo", "k_hi", "flags", "a_store", "b_store"],
    "formats": ["<i8", "<i8", "<i4", "<i4", "<i2", "<i2", "u1", "u1", "u1"],
    "offsets": [0, 8, 16, 20, 24, 26, 28, 29, 30],
    "itemsize": 32,
})
STORE = {0: "A", 1: "L", 2: "P1", 3: "S", 5: "T", 255: "-"}


def load(path):
    with open(path, "rb") as f:
        hdr = np.frombuffer(f.read(88), np.int64)
        if hdr[0] != -4:
            raise SystemExit(f"{path}: old trace format")
        ntask, batch, nq0, nb, ndep, nsig, nseg, ntiles, bp, nchain = (int(x) for x in hdr[1:])
        tasks = np.frombuffer(f.read(DTASK.itemsize * ntask), DTASK)
        deps = np.frombuffer(f.read(8 * ndep), DEP)
        sigs = np.frombuffer(f.read(4 * nsig), np.int32)
        segs = np.frombuffer(f.read(32 * nseg), SEG)
        tiles = np.frombuffer(f.read(8 * ntiles), np.int32).reshape(-1, 2)
        chain_tasks = np.frombuffer(f.read(DTASK.itemsize * nchain), DTASK)
        rec = np.frombuffer(f.read(), np.uint64).reshape(-1, 4)
    chain = rec[ntask * batch:]
    rec = rec[:ntask * batch]
    hchain = None
    if len(chain) == 2 * nchain * batch:  # eight-warp chain: worker 1's records follow
        chain, hchain = chain[:nchain * batch], chain[nchain * batch:]
    return dict(chain=chain, hchain=hchain, chain_tasks=chain_tasks,ntask=ntask, batch=batch, nq0=nq0, nb=nb, tasks=tasks, deps=deps, sigs=sigs, segs=segs, rec=rec,
                tiles=tiles, bp=bp)


def where(t, tiles, bp):
    """(tile i, tile j, block p, block q) of a task's output block, or the leaf's block."""
    off = int(t["c0_off"] if t["kind"] == 1 else t["c_off"])
    if t["c_store"] in (5,) and t["kind"] != 1:  # scratch: T blocks, per column j
        j, rem = divmod(off, bp * bp)
        return ("T", j, rem // bp // 64, rem % bp // 64)
    slot, rem = divmod(off, bp * bp)
    if slot >= len(tiles):
        return ("?", slot, 0, 0)
    i, j = tiles[slot]
    return (int(i), int(j), rem // bp // 64, rem % bp // 64)


def label(t, q0):
    if t["kind"] == 1:
        return "leaf" + ("+fat" if t["mode"] & 2 else "")
    if t["kind"] == 2:
        sp = f"/split{int(t['aux1']) & 255}"
    else:
        sp = ""
    cs, c0 = STORE.get(int(t["c_store"]), "?"), STORE.get(int(t["c0_store"]), "?")
    q = "q0" if q0 else "q1"
    name = {("q0", "L"): "paneld", ("q0", "A"): "traild", ("q0", "T"): "trow", ("q0", "P1"): "xrow",
            ("q1", "L"): "panel", ("q1", "A"): "update", ("q1", "P1"): "W"}.get((q, cs))
    if name is None:
        if cs == "S":
            name = {0: "off", 1: "symdiag", 2: "mirror"}[int(t["mode"])] + ("+c0" if c0 == "S" else "")
        else:
            name = f"{cs}"
    return f"{q}:{name}/s{int(t['seg_count'])}{sp}"


def chain_report(d, t0):
    ch = d["chain"].astype(np.float64) / 1e3
    if len(ch) == 0:
        return
    ok = ch[:, 0] > 0
    ch = ch[ok] - t0
    start, met, core, fat = ch[:, 0], ch[:, 1], ch[:, 2], ch[:, 3]
    n = len(ch)
    dep_wait = met - start
    core_t = core - met
    fat_wait = np.where(fat > 0, fat - core, 0)
    nxt = np.append(start[1:], np.nan)
    tail = nxt - core  # from core done (and fat) to the next step start
    print(f"  chain: {n} steps over {start[0]:.1f}..{core[-1]:.1f} us")
    print(f"    per step mean: dep wait {dep_wait.mean():.2f} us, leaf core {core_t.mean():.2f} (p50 {np.median(core_t):.2f}), "
          f"fat-phase wait {fat_wait.mean():.2f}, fat+rest {np.nanmean(tail - fat_wait):.2f}; step {np.nanmean(nxt - start):.2f} us")
    for a, b in ((0, 16), (16, 64), (64, 256), (n // 2, n // 2 + 200), (n - 64, n)):
        seg = slice(a, min(b, n))
        print(f"    steps {a}-{min(b, n)}: leaf core mean {core_t[seg].mean():.2f} us, step {np.nanmean((nxt - start)[seg]):.2f} us")
    nb = d["nb"]
    pos = np.arange(n) % nb
    for k in range(nb):
        m = pos == k
        print(f"    block {k} of the tile: leaf core {core_t[m].mean():.2f} us, fat wait {fat_wait[m].mean():.2f}, "
              f"rest to next step {np.nanmean((nxt - core - fat_wait)[m]):.2f}, step {np.nanmean((nxt - start)[m]):.2f}")
    if d.get("hchain") is not None and d["hchain"][:, 0].any():
        hc = d["hchain"].astype(np.float64)[ok] / 1e3 - t0
        s0, s1, s2, s3 = hc[:, 0], hc[:, 1], hc[:, 2], hc[:, 3]
        has2 = hc[:, 2] > 0
        print(f"    worker 1: S0 seen {np.mean(s0 - core):+.2f} us after the leaf, stores {np.mean(s1 - s0):.2f}, "
              f"S2 seen {np.mean((s2 - s1)[has2]):.2f} after, 2nd signals {np.mean((s3 - s2)[has2]):.2f}; "
              f"S1 published {np.nanmean(nxt - s1):.2f} us before the next step")
    first = np.arange(n) % nb == 0
    if first.any():
        print(f"    tile-first steps: dep wait mean {dep_wait[first].mean():.2f} us (total {dep_wait[first].sum() / 1e3:.1f} ms); "
              f"other steps dep wait total {dep_wait[~first].sum() / 1e3:.1f} ms, fat waits total {fat_wait.sum() / 1e3:.1f} ms")


def chain_deps_report(d, events, t0):
    """For the chain's boundary steps (mode 4): when each second-phase dependency
    was satisfied, relative to the end of the step's first phase."""
    ch = d["chain"].astype(np.float64) / 1e3
    if len(ch) == 0:
        return
    tasks_chain = d.get("chain_tasks")
    if tasks_chain is None:
        return
    deps = d["deps"]
    lat = {}
    nb = d["nb"]
    for si, st in enumerate(tasks_chain):
        if ch[si, 2] <= 0:
            continue
        core_end = ch[si, 2] - t0
        for k in range(st["dep_begin"] + st["dep_count"], st["dep_begin"] + st["dep_count"] + st["dep2_count"]):
            dp = deps[k]
            ev = events.get((int(dp["counter"]), 0), [])
            if dp["value"] > 0 and len(ev) >= dp["value"]:
                key = ("boundary" if st["mode"] & 4 else f"block{si % nb}", k - st["dep_begin"] - st["dep_count"])
                lat.setdefault(key, []).append(ev[dp["value"] - 1][0] - core_end)
    for k, v in sorted(lat.items()):
        v = np.array(v)
        print(f"    {k[0]} dep2[{k[1]}] satisfied {v.mean():+.1f} us after the leaf (p50 {np.median(v):+.1f}, max {v.max():+.1f})")
    # the producer chain behind the boundary's late second-phase dependencies,
    # for one boundary step in the middle of the sweep
    ctx = d.get("_ctx")
    bsteps = [si for si, st in enumerate(tasks_chain) if st["mode"] & 4 and ch[si, 2] > 0]
    if not bsteps or ctx is None:
        return
    for si in (bsteps[len(bsteps) // 2], bsteps[len(bsteps) // 2] - 4):
        walk_step(d, events, ctx, tasks_chain, ch, si, t0)


def walk_step(d, events, ctx, tasks_chain, ch, si, t0):
    deps = d["deps"]
    st = tasks_chain[si]
    core_end = ch[si, 2] - t0
    print(f"    chain step {si} (mode {int(st['mode'])}): producers of its second-phase deps (us relative to its leaf end):")
    for k in range(st["dep_begin"] + st["dep_count"], st["dep_begin"] + st["dep_count"] + st["dep2_count"]):
        dp = deps[k]
        ev = events.get((int(dp["counter"]), 0), [])
        if dp["value"] <= 0 or len(ev) < dp["value"]:
            continue
        r = ev[dp["value"] - 1][1]
        print(f"     dep2[{k - st['dep_begin'] - st['dep_count']}]:")
        for _ in range(6):
            t = d["tasks"][ctx["tidx"][r]]
            print(f"       {ctx['lab'][r]:24s} {str(where(t, d['tiles'], d['bp'])):22s} pushed {ctx['pushed'][r] - core_end:+8.1f} "
                  f"claim {ctx['claim'][r] - core_end:+8.1f} done {ctx['done'][r] - core_end:+8.1f}")
            best, bt, bchain = None, -1e18, False
            for kk in range(t["dep_begin"], t["dep_begin"] + t["dep_count"] + t["dep2_count"]):
                q = deps[kk]
                e = events.get((int(q["counter"]), 0), [])
                if q["value"] <= 0:
                    continue
                if len(e) < q["value"]:
                    bchain = True  # produced by a chain step (not in the task records)
                    continue
                if e[q["value"] - 1][0] > bt:
                    best, bt = e[q["value"] - 1][1], e[q["value"] - 1][0]
            if best is None:
                print("       <- chain step" if bchain else "       <- (start)")
                break
            if bchain:
                print(f"         (also waits on a chain step)")
            r = best


def report(path):
    d = load(path)
    tasks, deps, sigs, rec, batch, nq0 = d["tasks"], d["deps"], d["sigs"], d["rec"], d["batch"], d["nq0"]
    ok = rec[:, 2] > 0
    rec = rec[ok]
    claim, pushed, done = (rec[:, i].astype(np.float64) / 1e3 for i in range(3))  # us
    # v3 traces: field 1 = time the task was pushed to a ready queue (0: ready at start)
    ready = claim.copy()
    tidx = (rec[:, 3] >> 32).astype(np.int64)
    mat = ((rec[:, 3] >> 16) & 0xFFFF).astype(np.int64)
    sm = (rec[:, 3] & 0xFFFF).astype(np.int64)
    t0 = claim.min()
    pushed = np.where(pushed > 0, pushed, claim.min() * 1e0)
    claim, ready, done, pushed = claim - t0, ready - t0, done - t0, pushed - t0
    span = done.max()
    q0 = tidx < nq0
    labels = np.array([label(tasks[i], i < nq0) for i in range(len(tasks))])
    lab = labels[tidx]
    print(f"{path}: tasks={len(rec)} (q0 {q0.sum()}, q1 {(~q0).sum()}) batch={batch} span={span:.1f} us")
    chain_report(d, t0 / 1e0)
    nsm = len(np.unique(sm))
    busy_all = (done - ready).sum()
    print(f"  CTA-busy fraction {busy_all / (span * 2 * nsm):.3f} (2 CTAs x {nsm} SMs)")
    for name, m in (("q0/crit", q0), ("q1/bulk", ~q0)):
        if m.sum() == 0:
            continue
        wait = (ready[m] - claim[m]).sum()
        busy = (done[m] - ready[m]).sum()
        print(f"  {name}: busy {busy:.0f} us, waiting {wait:.0f} us (wait share {wait / (wait + busy):.2f}), "
              f"SMs {len(np.unique(sm[m]))}, last-done {done[m].max():.1f} us")
    dur = done - ready
    print("  per class: n, mean us, p50, total ms")
    for L in sorted(set(lab.tolist())):
        m = lab == L
        print(f"    {L:28s} n={m.sum():6d} mean {dur[m].mean():7.1f} p50 {np.median(dur[m]):7.1f} total {dur[m].sum() / 1e3:8.1f}")
    edges = np.linspace(0, span, 11)
    busy_t = []
    for a, b in zip(edges[:-1], edges[1:]):
        ov = np.clip(np.minimum(done, b) - np.maximum(ready, a), 0, None).sum()
        busy_t.append(ov / ((b - a) * 2 * nsm))
    print("  busy fraction per tenth of the sweep:", " ".join(f"{x:.2f}" for x in busy_t))

    # ---- critical path
    key = {(int(t), int(mm)): r for r, (t, mm) in enumerate(zip(tidx, mat))}
    events = collections.defaultdict(list)  # (counter, mat) -> [(done, rec)]
    # split groups signal once, through the reducer (the part that finished last)
    reducer = {}
    for r in range(len(rec)):
        t = tasks[tidx[r]]
        if t["kind"] == 2:
            g = (int(t["aux0"]), int(mat[r]))
            if g not in reducer or done[r] > done[reducer[g]]:
                reducer[g] = r
    for r in range(len(rec)):
        t = tasks[tidx[r]]
        if t["kind"] == 2 and reducer[(int(t["aux0"]), int(mat[r]))] != r:
            continue
        for s in range(t["sig_begin"], t["sig_begin"] + t["sig_count"]):
            events[(int(sigs[s]), int(mat[r]))].append((done[r], r))
    for v in events.values():
        v.sort()
    by_sm = collections.defaultdict(list)
    for r in np.argsort(done):
        by_sm[int(sm[r])].append(r)
    sm_done = {s: np.array([done[r] for r in rs]) for s, rs in by_sm.items()}
    # queue wait: claim time minus the time the task was pushed ready
    qwait = claim - pushed
    for name, m in (("q0", q0), ("q1", ~q0)):
        w = qwait[m]
        if len(w):
            print(f"  {name} queue wait (claim - pushed): mean {w.mean():.2f} us, p50 {np.median(w):.2f}, p90 "
                  f"{np.percentile(w, 90):.2f}, max {w.max():.1f}")
    d["_ctx"] = dict(tidx=tidx, lab=lab, pushed=pushed, claim=claim, done=done)
    chain_deps_report(d, events, t0)
    r = int(np.argmax(done))
    path_seq = []
    path_exec = collections.Counter()
    path_n = collections.Counter()
    gap_dep = gap_claim = 0.0
    steps = 0
    while r is not None and steps < 10 ** 7:
        steps += 1
        t = tasks[tidx[r]]
        path_seq.append(r)
        path_exec[lab[r]] += done[r] - ready[r]
        path_n[lab[r]] += 1
        best, bt = None, -1.0
        for k in range(t["dep_begin"], t["dep_begin"] + t["dep_count"] + t["dep2_count"]):
            dp = deps[k]
            ev = events.get((int(dp["counter"]), int(mat[r])), [])
            if dp["value"] <= 0 or len(ev) < dp["value"]:
                continue
            tm, pr = ev[dp["value"] - 1]
            if tm > bt:
                best, bt = pr, tm
        if best is None:
            break
        # queue wait before the claim (or second-phase wait inside the task)
        gap_claim += max(0.0, claim[r] - bt)
        r = best
    tot = sum(path_exec.values())
    print(f"  critical path: {sum(path_n.values())} tasks, exec {tot / 1e3:.1f} ms, "
          f"queue waits {gap_claim / 1e3:.1f} ms (span {span / 1e3:.1f} ms)")
    for L, v in path_exec.most_common():
        if path_n[L]:
            print(f"    {L:28s} n={path_n[L]:6d} exec {v / 1e3:8.2f} ms  mean {v / path_n[L]:6.1f} us")
    # a window of the path from the middle of the sweep, in time order
    seq = path_seq[::-1]
    mid = len(seq) // 2
    print("  critical path sample (claim, ready, done us; class; tile i, j; block p, q):")
    prev_done = None
    for r in seq[mid:mid + 60]:
        t = tasks[tidx[r]]
        w = where(t, d["tiles"], d["bp"])
        gap = "" if prev_done is None else f" (+{ready[r] - prev_done:.1f})"
        print(f"    {claim[r]:10.1f} {ready[r]:10.1f} {done[r]:10.1f}{gap:>9s}  {lab[r]:26s} {w}")
        prev_done = done[r]


if __name__ == "__main__":
    for p in sys.argv[1:]:
        report(p)
