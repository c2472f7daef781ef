"""CPU ORACLE (test infrastructure only) -- symbolic half + ctypes glue.

Restates the reference's symbolic analysis in pure Python (small tile grids:
N <= a few hundred) and drives the C restatement of the numeric kernels in
oracle/tileinv_oracle.c (liborc.so).  Only tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline leg import this module, and only as the CHECKER; the
product path (paper_2504_19171_b200) never touches it.

Parity of this oracle is pinned in tests/test_oracle.py against the reference
itself (oracle/_ref, built from /root/reference/proj by oracle/Makefile) and
the reference's known-answer tests (tests/golden/).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(HERE, "liborc.so")


def _load():
    if not os.path.exists(_LIB_PATH):
        subprocess.run(["make", "-s", "c_oracle"], cwd=HERE, check=True)
    lib = C.CDLL(_LIB_PATH)
    P = C.c_void_p
    lib.orc_generate_mask.argtypes = [C.c_long, C.c_long, C.c_long, C.c_double, C.c_uint64, C.c_int, C.c_int, P]
    lib.orc_generate_fill.argtypes = [C.c_long, C.c_long, C.c_long, C.c_double, C.c_uint64, C.c_int, C.c_int,
                                      P, P, P]
    lib.orc_factorize.argtypes = [C.c_int, C.c_int, P, P, P]
    lib.orc_factorize.restype = C.c_long
    lib.orc_logdet.argtypes = [C.c_int, C.c_int, C.c_long, P, P]
    lib.orc_logdet.restype = C.c_double
    lib.orc_phase1.argtypes = [C.c_int, C.c_int, P, P]
    lib.orc_phase2.argtypes = [C.c_int, C.c_int, P, P, P, P, P, P, P, C.c_long]
    lib.orc_phase2.restype = C.c_int
    return lib


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = _load()
    return _lib


def _ptr(a: np.ndarray):
    return C.c_void_p(a.ctypes.data)


# ---- symbolic analysis -------------------------------------------------------

def layout(n: int, b: int):
    """build_layout, proj/src/layout.cpp:11-20."""
    N = (n + b - 1) // b
    return N, N * b


def sort_tiles(tiles):
    """TilePattern ctor order, layout.cpp:36-53: column-major, deduplicated."""
    return sorted(set(tiles), key=lambda t: (t[1], t[0]))


def csc(N: int, tiles):
    cs = np.zeros(N + 1, np.int64)
    for _, j in tiles:
        cs[j + 1] += 1
    cs = np.cumsum(cs).astype(np.int64)
    rows = np.array([i for i, _ in tiles], np.int32)
    return cs, rows


def symbolic_fill(N: int, tiles):
    """layout.cpp:62-87: one ascending pass of the elimination closure."""
    cols = [set() for _ in range(N)]
    for i, j in tiles:
        cols[j].add(i)
    for k in range(N):
        below = sorted(r for r in cols[k] if r > k)
        for a in range(len(below)):
            for c in range(a, len(below)):
                cols[below[a]].add(below[c])
    return [(i, j) for j in range(N) for i in sorted(cols[j])]


def select_tiles(n: int, b: int, N: int, factor_tiles, selection):
    """selinv.cpp:51-83."""
    if selection == "diagonal":
        return [(i, i) for i in range(N)]
    if selection == "pattern":
        return list(factor_tiles)
    if selection == "all":
        return [(i, j) for j in range(N) for i in range(j, N)]
    out = []
    for r, c in selection:
        if r < 0 or c < 0 or r >= n or c >= n:
            raise ValueError(f"requested entry ({r}, {c}) outside the matrix")
        r, c = max(r, c), min(r, c)
        out.append((r // b, c // b))
    return sort_tiles(out)


def symbolic_inversion(N: int, requested, factor_tiles):
    """selinv.cpp:85-150: closure + per-column work (columns descending,
    off-diagonal rows descending)."""
    nb = [[] for _ in range(N)]
    for i, j in factor_tiles:
        nb[j].append(i)
    col_rows = [set() for _ in range(N)]
    for i, j in sort_tiles(requested):
        col_rows[j].add(i)
    for i in range(N):
        rows = col_rows[i]
        if not rows:
            continue
        if i in rows:
            rows.update(k for k in nb[i] if k > i)
        for r in sorted(rows):
            if r <= i:
                continue
            for k in nb[i]:
                if k > i:
                    col_rows[min(r, k)].add(max(r, k))
    closure = [(r, i) for i in range(N) for r in sorted(col_rows[i])]
    work = []
    for i in range(N - 1, -1, -1):
        rows = col_rows[i]
        if not rows:
            continue
        off = sorted((r for r in rows if r > i), reverse=True)
        work.append((i, i in rows, off))
    return closure, work


# ---- numeric drivers --------------------------------------------------------

def generate(n, w, t, density, seed, b):
    """generate_arrowhead, matgen.cpp:59-120 -> (N, tiles, payload[T,b,b])."""
    N, _ = layout(n, b)
    mask = np.zeros(N * N, np.uint8)
    lib().orc_generate_mask(n, w, t, float(density), seed, b, N, _ptr(mask))
    mask = mask.reshape(N, N)
    tiles = [(i, j) for j in range(N) for i in range(j, N) if mask[i, j]]
    cs, rows = csc(N, tiles)
    pay = np.zeros((len(tiles), b, b))
    lib().orc_generate_fill(n, w, t, float(density), seed, b, N, _ptr(cs), _ptr(rows), _ptr(pay))
    return N, tiles, pay


def tiles_from_dense(a: np.ndarray, b: int):
    """from_dense, module.cpp:46-74."""
    n = a.shape[0]
    N, npad = layout(n, b)
    blocks = {}
    for r in range(n):
        for c in range(r + 1):
            v = a[r, c]
            if v == 0.0 and r != c:
                continue
            blocks.setdefault((r // b, c // b), np.zeros((b, b)))[r % b, c % b] = v
    for i in range(N):
        blocks.setdefault((i, i), np.zeros((b, b)))
    for r in range(n, npad):
        blocks[(r // b, r // b)][r % b, r % b] = 1.0
    tiles = sort_tiles(blocks)
    return N, tiles, np.stack([blocks[t] for t in tiles])


def selected_inverse(n, b, N, tiles, payload, selection="pattern"):
    """selected_inverse(matrix, request) (selinv.cpp:359-367): factorize ->
    select -> closure -> phase1 -> phase2.  Returns a dict with the closure
    tiles, Sigma payload, diag(Sigma) (when the diagonal is in the closure),
    logdet, the factor tiles and the phase-1 tiles."""
    filled = symbolic_fill(N, tiles)
    fcs, frows = csc(N, filled)
    src = {t: k for k, t in enumerate(tiles)}
    pay = np.zeros((len(filled), b, b))
    for k, t in enumerate(filled):
        if t in src:
            pay[k] = payload[src[t]]
    bad = lib().orc_factorize(N, b, _ptr(fcs), _ptr(frows), _ptr(pay))
    if bad != -1:
        return {"not_spd_pivot": int(bad)}
    L = pay.copy()
    logdet = lib().orc_logdet(N, b, n, _ptr(fcs), _ptr(pay))
    lib().orc_phase1(N, b, _ptr(fcs), _ptr(pay))
    req = select_tiles(n, b, N, filled, selection)
    closure, work = symbolic_inversion(N, req, filled)
    ccs, crows = csc(N, closure)
    flat = []
    for i, diag, off in work:
        flat += [i, int(diag), len(off)] + list(off)
    flat = np.array(flat, np.int32)
    sigma = np.zeros((len(closure), b, b))
    rc = lib().orc_phase2(N, b, _ptr(fcs), _ptr(frows), _ptr(pay), _ptr(ccs), _ptr(crows), _ptr(sigma),
                          _ptr(flat), len(flat))
    if rc != 0:
        raise RuntimeError("oracle phase 2: operand missing from closure")
    cidx = {t: k for k, t in enumerate(closure)}
    diag = None
    if all((i, i) in cidx for i in range(N)):
        diag = np.array([sigma[cidx[(r // b, r // b)], r % b, r % b] for r in range(n)])
    return {"tiles": closure, "payload": sigma, "diag": diag, "logdet": logdet, "factor_tiles": filled,
            "factor": L, "phase1": pay, "requested": req}


def selected_inverse_generated(n, w, t, density, seed, b, selection="pattern"):
    N, tiles, pay = generate(n, w, t, density, seed, b)
    return selected_inverse(n, b, N, tiles, pay, selection)


def entries_order(n, b, N, closure, requested, selection):
    """extract_entries order (selinv.cpp:387-439)."""
    if selection == "diagonal":
        return [(r, r) for r in range(n)]
    if selection == "all":
        return [(r, c) for c in range(n) for r in range(c, n)]
    if selection == "pattern":
        cols = [[] for _ in range(N)]
        for i, j in requested:
            cols[j].append(i)
        out = []
        for j in range(N):
            for oc in range(b):
                c = j * b + oc
                if c >= n:
                    break
                for i in cols[j]:
                    for orr in range(b):
                        r = i * b + orr
                        if r >= n:
                            break
                        if r >= c:
                            out.append((r, c))
        return out
    seen, out = set(), []
    for r, c in selection:
        if (r, c) in seen:
            continue
        seen.add((r, c))
        out.append((r, c))
    return out
