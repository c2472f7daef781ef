"""CPU interpreter of the device dataflow plans (test infrastructure).

Executes the task lists exported by `plan_export` with numpy block products,
claiming tasks strictly in order from the two queues the way
dataflow_kernel does (a reserved critical worker plus one bulk worker that
only takes a ready critical head): if neither queue head is ready the plan
would deadlock on the GPU, and the simulator raises.  This checks, without a
GPU, that the task decomposition, the operand addressing, the dependency
counters and the queue order reproduce the oracle's results.
"""
import numpy as np
from numpy.lib.stride_tricks import as_strided

K_STORE = {"A": 0, "L": 1, "P1": 2, "SIGMA": 3, "VAR": 4, "SCRATCH": 5, "LOGDET": 6, "STATUS": 7}
NONE = 255
TRANS_A, TRANS_B, NEGATE = 1, 2, 4
FULL, SYMDIAG, MIRROR = 0, 1, 2
BLK = 64


def view(flat, off, rows, cols, ld):
    base = flat[off:]
    return as_strided(base, shape=(rows, cols), strides=(ld * 8, 8))


class Sim:
    def __init__(self, plan, stores, status):
        self.p = plan
        self.s = stores
        self.cnt = np.zeros(plan["counters"], np.int64)
        self.status = status  # list with first bad pivot

    def ready(self, t):
        d = self.p["deps"][t["dep_begin"]:t["dep_begin"] + t["dep_count"] + t["dep2_count"]]
        return all(self.cnt[c] >= v for c, v in zip(d["counter"], d["value"]))

    def gemm(self, t):
        """Block GEMM task; a split task (kind 2) stores its partial and only
        the last of its group reduces (in part order) and signals."""
        acc = self.product(t)
        if t["kind"] == 2:
            part, parts = int(t["aux1"]) >> 8, int(t["aux1"]) & 255
            slots = self.s[K_STORE["SCRATCH"]]
            base = int(t["p_off"])
            slots[base + part * BLK * BLK: base + (part + 1) * BLK * BLK] = acc.reshape(-1)
            self.cnt[int(t["aux0"])] += 1
            if self.cnt[int(t["aux0"])] < parts:
                return False
            acc = slots[base: base + parts * BLK * BLK].reshape(parts, BLK, BLK)[0].copy()
            for q in range(1, parts):
                acc = acc + slots[base + q * BLK * BLK: base + (q + 1) * BLK * BLK].reshape(BLK, BLK)
        self.epilogue(t, acc)
        return True

    def product(self, t):
        acc = np.zeros((BLK, BLK))
        for g in self.p["segs"][t["seg_begin"]:t["seg_begin"] + t["seg_count"]]:
            klo, khi = int(g["k_lo"]), int(g["k_hi"])
            if khi <= klo:
                continue
            A, B = self.s[int(g["a_store"])], self.s[int(g["b_store"])]
            m0, n0, lda, ldb = int(t["m0"]), int(t["n0"]), int(g["lda"]), int(g["ldb"])
            if g["flags"] & TRANS_A:
                opa = view(A, int(g["a_off"]) + klo * lda + m0, khi - klo, BLK, lda).T
            else:
                opa = view(A, int(g["a_off"]) + m0 * lda + klo, BLK, khi - klo, lda)
            if g["flags"] & TRANS_B:
                opb = view(B, int(g["b_off"]) + n0 * ldb + klo, BLK, khi - klo, ldb).T
            else:
                opb = view(B, int(g["b_off"]) + klo * ldb + n0, khi - klo, BLK, ldb)
            prod = opa @ opb
            acc += -prod if g["flags"] & NEGATE else prod
        return acc

    def epilogue(self, t, acc):
        ldc = int(t["ldc"])
        if t["c0_store"] != NONE:
            acc = acc + view(self.s[int(t["c0_store"])], int(t["c0_off"]), BLK, BLK, int(t["ldc0"]))
        C = view(self.s[int(t["c_store"])], int(t["c_off"]), BLK, BLK, ldc)
        mode = int(t["mode"])
        if mode == FULL:
            C[:] = acc
        elif mode == MIRROR:
            C[:] = acc
            view(self.s[int(t["cm_store"])], int(t["cm_off"]), BLK, BLK, ldc)[:] = acc.T
        else:
            low = np.tril(acc)
            C[:] = low + np.tril(acc, -1).T
            if t["diag_store"] != NONE:
                self.s[int(t["diag_store"])][int(t["diag_off"]):int(t["diag_off"]) + BLK] = np.diag(acc)

    def leaf(self, t):
        ld = int(t["ldc"])
        A = view(self.s[K_STORE["A"]], int(t["c_off"]), BLK, BLK, int(t["ldc0"]))
        # (the upper blocks of the diagonal tiles are cleared by the zero-strip
        # kernel on the GPU; the simulator's stores start zeroed)
        Lv = view(self.s[K_STORE["L"]], int(t["c0_off"]), BLK, BLK, ld)
        Xv = view(self.s[K_STORE["P1"]], int(t["cm_off"]), BLK, BLK, ld)
        a = np.tril(A)
        a = a + np.tril(a, -1).T
        valid = int(t["m0"])
        try:
            L = np.linalg.cholesky(a)
        except np.linalg.LinAlgError:
            piv = next(i for i in range(BLK) if not np.all(np.linalg.eigvalsh(a[: i + 1, : i + 1]) > 0))
            if piv < valid:
                self.status[0] = min(self.status[0], int(t["n0"]) + piv)
            L = np.full((BLK, BLK), np.nan)
        X = np.linalg.inv(L) if np.all(np.isfinite(L)) else L
        Lv[:, :BLK] = np.tril(L)
        Xv[:, :BLK] = np.tril(X)
        self.s[K_STORE["LOGDET"]][int(t["diag_off"])] = np.sum(np.log(np.diag(L)[: max(0, valid)]))
        if t["mode"] & 4:  # tile-boundary leaf: (P - S_0) X^T and the next diagonal block's last term
            g = self.p["segs"][int(t["seg_begin"])]
            S = view(self.s[int(g["a_store"])], int(g["a_off"]), BLK, BLK, int(g["lda"]))
            P = view(self.s[K_STORE["A"]], int(t["p_off"]), BLK, BLK, ld)
            Lp = (P - S) @ np.tril(X).T
            view(self.s[K_STORE["L"]], int(t["p_off"]), BLK, BLK, ld)[:] = Lp
            D = view(self.s[int(g["b_store"])], int(g["b_off"]), BLK, BLK, ld)
            D[:] = D - np.tril(Lp @ Lp.T)
        if t["mode"] & 2:  # fat leaf: next panel block and diagonal update
            P = view(self.s[K_STORE["A"]], int(t["c_off"]) + BLK * ld, BLK, BLK, ld)
            Lp = P @ np.tril(X).T
            view(self.s[K_STORE["L"]], int(t["c0_off"]) + BLK * ld, BLK, BLK, ld)[:] = Lp
            D = view(self.s[K_STORE["A"]], int(t["c_off"]) + BLK * ld + BLK, BLK, BLK, ld)
            D[:] = D - np.tril(Lp @ Lp.T)

    def run(self):
        tasks = self.p["tasks"]
        q = [list(range(self.p["q0"])), list(range(self.p["q0"], len(tasks)))]
        head = [0, 0]
        while head[0] < len(q[0]) or head[1] < len(q[1]):
            for qi in (0, 1):
                if head[qi] < len(q[qi]) and self.ready(tasks[q[qi][head[qi]]]):
                    t = tasks[q[qi][head[qi]]]
                    head[qi] += 1
                    break
            else:
                raise RuntimeError(f"dataflow deadlock: heads {head}")
            if t["kind"] == 1:
                self.leaf(t)
            elif not self.gemm(t):
                continue
            sg = self.p["sigs"][t["sig_begin"]:t["sig_begin"] + t["sig_count"]]
            np.add.at(self.cnt, sg, 1)


    def run_random(self, seed):
        """Executes the tasks one at a time in a random order among those whose
        dependencies (both phases) are met -- the GPU may run any ready task at
        any time, so a dependency missing from the plan shows up as a wrong
        result here for some seed."""
        rng = np.random.default_rng(seed)
        tasks = self.p["tasks"]
        deps = self.p["deps"]
        waiters = {}
        missing = np.zeros(len(tasks), np.int64)
        for ti, t in enumerate(tasks):
            d = deps[t["dep_begin"]:t["dep_begin"] + t["dep_count"] + t["dep2_count"]]
            for c, v in zip(d["counter"].tolist(), d["value"].tolist()):
                if v > self.cnt[c]:
                    missing[ti] += 1
                    waiters.setdefault((c, v), []).append(ti)
        ready = [ti for ti in range(len(tasks)) if missing[ti] == 0]
        done = 0
        while ready:
            k = int(rng.integers(len(ready)))
            ti = ready[k]
            ready[k] = ready[-1]
            ready.pop()
            done += 1
            t = tasks[ti]
            if t["kind"] == 1:
                self.leaf(t)
            elif not self.gemm(t):
                continue
            for c in self.p["sigs"][t["sig_begin"]:t["sig_begin"] + t["sig_count"]].tolist():
                self.cnt[c] += 1
                for w in waiters.pop((c, int(self.cnt[c])), []):
                    missing[w] -= 1
                    if missing[w] == 0:
                        ready.append(w)
        if done != len(tasks):
            raise RuntimeError(f"dataflow deadlock: {done} of {len(tasks)} tasks ran")


def run_plans(tib, matrix, selection, order=None, split=-1, batch=1):
    """Runs factor + phase-2 plans of `matrix` on the CPU interpreter (in-order
    queue claiming, or a random ready order seeded by `order`; split > 0: the
    two-chain factor plan); returns (factor tiles, closure tiles, Sigma payload
    [T, b, b], logdet, first bad pivot)."""
    fpat = tib.factor_pattern(matrix)
    closure, _ = tib.closure_tiles(matrix, selection)
    pf = tib.plan_export(matrix, selection, 0, crit_workers=1, split=split, batch=batch)
    pp = tib.plan_export(matrix, selection, 1, crit_workers=1, split=split, batch=batch)
    bp, b, n = pf["bp"], matrix.tile_size, matrix.n
    N = matrix.n_tiles
    nb = bp // BLK
    ti, tj, pay = matrix.tiles()
    src = {(int(i), int(j)): k for k, (i, j) in enumerate(zip(ti, tj))}
    A = np.zeros((len(fpat), bp, bp))
    for k, (i, j) in enumerate(fpat):
        if (i, j) in src:
            A[k, :b, :b] = pay[src[(i, j)]]
        if i == j:
            A[k, b:, b:] = np.eye(bp - b)
    stores = {
        0: A.reshape(-1).copy(),
        1: np.zeros(len(fpat) * bp * bp),
        2: np.zeros(len(fpat) * bp * bp),
        3: np.zeros(len(closure) * bp * bp),
        4: np.zeros(N * bp),
        5: np.zeros(max(pf["scratch_doubles"], pp["scratch_doubles"], 1)),
        6: np.zeros(N * nb),
    }
    status = [np.iinfo(np.int64).max]
    for plan in (pf, pp):
        sim = Sim(plan, stores, status)
        if order is None:
            sim.run()
        else:
            sim.run_random(order)
    sig = stores[3].reshape(len(closure), bp, bp)[:, :b, :b]
    logdet = 2.0 * stores[6].sum()
    return fpat, closure, sig, logdet, status[0], stores[4].reshape(N, bp)[:, :b].reshape(-1)[:n]
