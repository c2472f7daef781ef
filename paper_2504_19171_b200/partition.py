"""Partitioned single-matrix path: one band+arrow
matrix split into tile-column blocks, one block per GPU, with the separator
and arrow-block Schur contributions reduced over NVLink (NCCL all-reduce).

The reference has no partitioned mode (its elimination order is a sequential
column chain, "future work"), so this is an ordering change, not
a restatement: L differs from the reference's, but Sigma on the matrix's own
tile pattern, the marginal variances and the log-determinant are invariant
under the symmetric permutation and are checked against the oracle.

Ordering.  The band columns 0 .. N-2 are cut into P interiors I_0 .. I_{P-1}
separated by P-1 separators S_0 .. S_{P-2} of `sep` = band-width tile columns
each (no band tile connects I_p with I_q, p != q); the arrow tile row N-1 is
last.  Global order: [I_0, .., I_{P-1}, S_0, .., S_{P-2}, arrow].  Rank p
owns the local system

    M_p = [[A_II, A_IB], [A_BI, A_BB]],   I = I_p,  B = B_p = [S_{p-1}, S_p, arrow]

in the local order [I_p, S_{p-1}, S_p, arrow] (a band+arrow matrix whose
arrow is the border; S_{p-1} fills in across I_p, so ranks p >= 1 carry a
thicker arrow and get fewer columns, `weights`).

  A  factorize M_p (fused device sweep): L_II, L_BI, L_BB with
     L_BB L_BB^T = A_BB - C_p,  C_p = A_BI A_II^{-1} A_IB = A_BB - L_BB L_BB^T.
  B  all-reduce (NCCL) of the C_p scattered into the reduced system over
     R = [S_0, .., S_{P-2}, arrow]:  S = A_RR - sum_p C_p (the Schur
     complement of every interior).
  C  selected inversion of S (replicated on every rank; block-tridiagonal
     separators + arrow): Sigma_RR on its pattern, logdet(S).
  D  E_p = Sigma_{B_p B_p};  M_p' = M_p with A_BB replaced by E_p^{-1} + C_p
     has the factor [L_II, L_BI, chol(E_p^{-1})] -- only the border tiles of the
     phase-A factor change (Factor.replace_tiles) -- and
     (M_p'^{-1})_{II} = A_II^{-1} + A_II^{-1} A_IB E_p A_BI A_II^{-1} = Sigma_II,
     (M_p'^{-1})_{BI} = Sigma_{B_p I_p}:  the selected inverse of the modified
     factor gives the global Sigma on the interior and its border couplings.
  logdet(A) = sum_p [logdet(M_p) - logdet(L_BB L_BB^T)] + logdet(S).

The orchestration is written against an `engine` (the device library here;
tests/partition_sim.py supplies a dense numpy one, the CPU prototype) and an
`allreduce` (torch.distributed over NCCL on GPUs, gloo on CPU, or the
identity when one process runs every part).
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np


@dataclass
class BandArrowPartition:
    """Tile-column partition of an N-tile band+arrow grid over P parts."""

    N: int           # tile columns of the matrix
    band: int        # largest i - j of a band (non-arrow) tile
    parts: int
    arrow_tiles: int = 1  # trailing dense tile rows (the arrow; two when it straddles a tile boundary)
    weights: list = field(default=None)  # relative work per interior column of each part

    def __post_init__(self):
        P, s = self.parts, self.band
        if P < 1:
            raise ValueError("need at least one part")
        if s < 1 and P > 1:
            raise ValueError("a partition needs a band of at least one tile")
        na = self.arrow_tiles
        ncols = self.N - na  # band columns
        free = ncols - (P - 1) * s
        if P > 1 and free < P * max(s, 1):
            raise ValueError(f"{ncols} band tile columns cannot hold {P} interiors of >= {s} tiles "
                             f"and {P - 1} separators of {s}")
        if self.weights is None:
            # a part with a left separator carries it as s more filled arrow
            # tiles per column: update work ~ (tiles per column)^2
            fill = ((2 * s + na) / (s + na)) ** 2
            self.weights = [1.0] + [fill] * (P - 1)
        inv = [1.0 / w for w in self.weights]
        raw = [free * x / sum(inv) for x in inv]
        sizes = [max(max(s, 1), int(math.floor(r))) for r in raw]
        # hand out the remainder to the parts with the largest fractional share
        while sum(sizes) < free:
            k = max(range(P), key=lambda q: raw[q] - sizes[q])
            sizes[k] += 1
        while sum(sizes) > free:
            k = max(range(P), key=lambda q: sizes[q] - raw[q] if sizes[q] > max(s, 1) else -1e9)
            sizes[k] -= 1
        self.interiors, self.seps = [], []
        c = 0
        for p in range(P):
            self.interiors.append(list(range(c, c + sizes[p])))
            c += sizes[p]
            if p < P - 1:
                self.seps.append(list(range(c, c + s)))
                c += s
        assert c == ncols
        self.arrow = list(range(ncols, self.N))
        self.last = self.N - 1  # the only tile that may be partial
        # reduced system R = [S_0, .., S_{P-2}, arrow]
        self.reduced = [t for sp in self.seps for t in sp] + self.arrow
        self.red_pos = {t: k for k, t in enumerate(self.reduced)}

    def border(self, p: int) -> list:
        b = []
        if p >= 1:
            b += self.seps[p - 1]
        if p <= self.parts - 2:
            b += self.seps[p]
        return b + self.arrow

    def local_order(self, p: int) -> list:
        """Global tile indices of part p in its local order [I_p, S_{p-1}, S_p, arrow]."""
        return self.interiors[p] + self.border(p)


def band_of(ti, tj, N: int) -> tuple[int, int]:
    """(band width, arrow tile rows) of a band+arrow tile set: the arrow is the
    longest suffix of full tile rows (every tile (i, j), j <= i, present), the
    band the largest i - j over the other tiles."""
    ti = np.asarray(ti)
    tj = np.asarray(tj)
    if np.count_nonzero(ti == tj) != N:
        raise ValueError("the pattern must hold every diagonal tile")
    per_row = np.bincount(ti, minlength=N)
    na = 0
    while na < N - 1 and per_row[N - 1 - na] == N - na:
        na += 1
    na = max(na, 1)
    non = ti < N - na
    bw = int((ti[non] - tj[non]).max()) if non.any() else 0
    return bw, na


class TileMap:
    """Host view of a symmetric tiled matrix: tile (i, j) for any i, j (upper
    tiles as transposes of the stored lower ones), scalar size per tile."""

    def __init__(self, n: int, b: int, ti, tj, pay):
        self.n, self.b = n, b
        self.N = (n + b - 1) // b
        self.pay = pay
        self.idx = {(int(i), int(j)): k for k, (i, j) in enumerate(zip(ti, tj))}

    def get(self, i: int, j: int):
        if i >= j:
            k = self.idx.get((i, j))
            return None if k is None else self.pay[k]
        k = self.idx.get((j, i))
        return None if k is None else self.pay[k].T

    def rows(self, t: int) -> int:
        return min(self.b, self.n - t * self.b)


def local_system(A: TileMap, order: list):
    """Tiles of A restricted to `order` (global tile indices, in local order):
    (n_local, ti, tj, payload).  Only the last tile may be partial (the arrow)."""
    b = A.b
    for t in order[:-1]:
        if A.rows(t) != b:
            raise ValueError("only the arrow tile may be partial")
    n_loc = (len(order) - 1) * b + A.rows(order[-1])
    ti, tj, pay = [], [], []
    for lj, gj in enumerate(order):
        for li in range(lj, len(order)):
            gi = order[li]
            if li == lj:
                t = A.get(gi, gi)
            else:
                t = A.get(gi, gj) if gi > gj else A.get(gj, gi)
                if t is not None and gi < gj:
                    t = t.T
            if t is not None:
                ti.append(li)
                tj.append(lj)
                pay.append(np.ascontiguousarray(t))
    return n_loc, np.array(ti, np.int32), np.array(tj, np.int32), np.stack(pay)


def dense_block(A_get, order: list, b: int, rows_last: int) -> np.ndarray:
    """Dense symmetric block over `order` (tile indices, the last one partial
    with rows_last rows) from a tile accessor A_get(i, j) -> b x b or None
    (lower tiles; diagonal tiles significant in their lower triangle)."""
    k = len(order)
    nd = (k - 1) * b + rows_last
    D = np.zeros((k * b, k * b))
    for lj in range(k):
        for li in range(lj, k):
            t = A_get(li, lj)
            if t is None:
                continue
            blk = np.asarray(t)
            if li == lj:
                blk = np.tril(blk)
                blk = blk + np.tril(blk, -1).T
                D[li * b:(li + 1) * b, lj * b:(lj + 1) * b] = blk
            else:
                D[li * b:(li + 1) * b, lj * b:(lj + 1) * b] = blk
                D[lj * b:(lj + 1) * b, li * b:(li + 1) * b] = blk.T
    return D[:nd, :nd]


def lower_tiles(Ld: np.ndarray, b: int, offset: int):
    """Lower tiles of a dense lower-triangular block, padded to whole tiles
    (identity on the padded diagonal), as (coords shifted by offset, payload)."""
    nd = Ld.shape[0]
    k = (nd + b - 1) // b
    full = np.zeros((k * b, k * b))
    full[:nd, :nd] = Ld
    for r in range(nd, k * b):
        full[r, r] = 1.0
    coords, pay = [], []
    for j in range(k):
        for i in range(j, k):
            coords.append((offset + i, offset + j))
            pay.append(full[i * b:(i + 1) * b, j * b:(j + 1) * b])
    return coords, np.stack(pay)


@dataclass
class PartResult:
    part: int
    sigma: dict          # (gi, gj) -> b x b tile of Sigma, original lower tiles touching the interior
    diag: np.ndarray     # marginal variances of the interior rows
    rows: np.ndarray     # their global scalar rows


@dataclass
class ReducedResult:
    sigma: np.ndarray    # dense Sigma_RR on the reduced system's pattern (zeros elsewhere)
    logdet: float
    order: list          # global tile indices of R


class DeviceEngine:
    """The library's device path for every numeric step."""

    def __init__(self, device: int = 0):
        import paper_2504_19171_b200 as tib

        self.tib = tib
        self.device = device

    def factorize(self, n, b, ti, tj, pay):
        m = self.tib.from_tiles(n, b, ti, tj, pay.reshape(len(ti), b, b))
        return self.tib.factorize(m, device=self.device)

    def factor_logdet(self, f) -> float:
        return f.logdet()

    def factor_tiles(self, f, coords):
        return f.get_tiles(coords)

    def gram(self, L: np.ndarray) -> np.ndarray:
        import torch

        t = torch.from_numpy(L).to(f"cuda:{self.device}")
        return (t @ t.T).cpu().numpy()

    def inverse(self, E: np.ndarray, b: int) -> np.ndarray:
        r = self.tib.selected_inverse(self.tib.from_dense(E, tile_size=b), "all", device=self.device)
        return r.to_dense()

    def cholesky(self, F: np.ndarray, b: int) -> np.ndarray:
        f = self.tib.factorize(self.tib.from_dense(F, tile_size=b), device=self.device)
        ti, tj, pay = f.tiles()
        n = F.shape[0]
        k = (n + b - 1) // b
        Ld = np.zeros((k * b, k * b))
        for i, j, t in zip(ti, tj, pay):
            Ld[i * b:(i + 1) * b, j * b:(j + 1) * b] = t
        return np.tril(Ld[:n, :n])

    def replace_and_invert(self, f, coords, tiles):
        f.replace_tiles(coords, tiles)
        r = self.tib.selected_inverse_of_factor(f, "pattern")
        ti, tj, pay = r.tiles()
        return {(int(i), int(j)): p for i, j, p in zip(ti, tj, pay)}, r.diagonal()

    def reduced_inverse(self, S: np.ndarray, b: int):
        r = self.tib.selected_inverse(self.tib.from_dense(S, tile_size=b), "pattern", device=self.device)
        return r.to_dense(), r.logdet()


def phase_a(A: TileMap, part: BandArrowPartition, p: int, engine):
    """Factor of rank p's local system and its Schur contribution C_p over its border."""
    b = A.b
    order = part.local_order(p)
    n_int = len(part.interiors[p])
    n_loc, ti, tj, pay = local_system(A, order)
    f = engine.factorize(n_loc, b, ti, tj, pay)
    nbt = len(order) - n_int
    coords = [(n_int + i, n_int + j) for j in range(nbt) for i in range(j, nbt)]
    Lt = engine.factor_tiles(f, coords)
    rows_last = A.rows(order[-1])
    L_BB = _dense_lower({c: t for c, t in zip(coords, Lt)}, n_int, nbt, b, rows_last)
    border = order[n_int:]
    D = dense_block(lambda i, j: A.get(border[i], border[j]) if border[i] >= border[j]
                    else _t(A.get(border[j], border[i])), list(range(nbt)), b, rows_last)
    C = D - engine.gram(L_BB)
    d = np.diag(L_BB)
    logdet_int = engine.factor_logdet(f) - 2.0 * float(np.log(d).sum())
    return f, C, L_BB, logdet_int


def _t(x):
    return None if x is None else x.T


def _dense_lower(lut, off, k, b, rows_last):
    n = (k - 1) * b + rows_last
    Ld = np.zeros((k * b, k * b))
    for (i, j), t in lut.items():
        Ld[(i - off) * b:(i - off + 1) * b, (j - off) * b:(j - off + 1) * b] = t
    return np.tril(Ld[:n, :n])


def scatter_reduced(part: BandArrowPartition, p: int, C: np.ndarray, b: int, rows_last: int,
                    out: np.ndarray) -> None:
    """Adds rank p's C_p (over its border, local order) into the dense reduced
    system `out` (over R)."""
    border = part.border(p)
    for a, ga in enumerate(border):
        ra = part.red_pos[ga]
        ha = rows_last if ga == part.last else b
        for c, gc in enumerate(border):
            rc = part.red_pos[gc]
            hc = rows_last if gc == part.last else b
            out[ra * b:ra * b + ha, rc * b:rc * b + hc] += C[a * b:a * b + ha, c * b:c * b + hc]


def reduced_matrix(A: TileMap, part: BandArrowPartition, G: np.ndarray) -> np.ndarray:
    """S = A_RR - G (dense over R)."""
    R = part.reduced
    rows_last = A.rows(part.last)
    ARR = dense_block(lambda i, j: A.get(R[i], R[j]) if R[i] >= R[j] else _t(A.get(R[j], R[i])),
                      list(range(len(R))), A.b, rows_last)
    return ARR - G


def phase_d(A: TileMap, part: BandArrowPartition, p: int, f, red: ReducedResult, engine) -> PartResult:
    """Border replaced by chol(E_p^{-1}), selected inverse of the modified factor."""
    b = A.b
    order = part.local_order(p)
    n_int = len(part.interiors[p])
    border = order[n_int:]
    rows_last = A.rows(part.last)
    idx = []
    for g in border:
        r = part.red_pos[g]
        idx.extend(range(r * b, r * b + (rows_last if g == part.last else b)))
    idx = np.asarray(idx)
    E = red.sigma[np.ix_(idx, idx)]
    F = engine.inverse(E, b)
    F = 0.5 * (F + F.T)
    LF = engine.cholesky(F, b)
    coords, tiles = lower_tiles(LF, b, n_int)
    sig, diag = engine.replace_and_invert(f, coords, tiles)
    out = {}
    interior = set(part.interiors[p])
    for (li, lj), t in sig.items():
        gi, gj = order[li], order[lj]
        if gi not in interior and gj not in interior:
            continue  # border x border: Sigma_RR holds it
        if gi >= gj:
            key, val = (gi, gj), t
        else:
            key, val = (gj, gi), t.T
        if A.get(*key) is None:
            continue  # fill-in tile: not in the matrix's own pattern
        out[key] = np.ascontiguousarray(val)
    rows = np.concatenate([np.arange(g * b, g * b + b) for g in part.interiors[p]])
    return PartResult(p, out, np.asarray(diag)[:n_int * b], rows)


def run(A: TileMap, part: BandArrowPartition, my_parts, engine, allreduce):
    """The four phases for the parts this process owns; returns (per-part
    results, reduced result, global logdet)."""
    b = A.b
    rows_last = A.rows(part.last)
    nR = (len(part.reduced) - 1) * b + rows_last
    G = np.zeros((nR, nR))
    state, ld_int = {}, 0.0
    for p in my_parts:
        f, C, _, ldi = phase_a(A, part, p, engine)
        scatter_reduced(part, p, C, b, rows_last, G)
        state[p] = f
        ld_int += ldi
    G, ld_int = allreduce(G, ld_int)
    S = reduced_matrix(A, part, G)
    S = 0.5 * (S + S.T)
    sig_R, ld_S = engine.reduced_inverse(S, b)
    red = ReducedResult(sig_R, ld_S, part.reduced)
    results = [phase_d(A, part, p, state[p], red, engine) for p in my_parts]
    return results, red, ld_int + ld_S


def assemble(A: TileMap, part: BandArrowPartition, results, red: ReducedResult):
    """Global Sigma tiles on A's own pattern, diag(Sigma) (every row), from the
    parts' results and the reduced result (test / gather helper)."""
    b = A.b
    sigma = {}
    diag = np.zeros(A.n)
    for r in results:
        sigma.update(r.sigma)
        diag[r.rows] = r.diag
    R = part.reduced
    rows_last = A.rows(part.last)
    for a, ga in enumerate(R):
        for c, gc in enumerate(R):
            if ga < gc or A.get(ga, gc) is None:
                continue
            blk = np.zeros((b, b))
            ha = rows_last if ga == part.last else b
            hc = rows_last if gc == part.last else b
            blk[:ha, :hc] = red.sigma[a * b:a * b + ha, c * b:c * b + hc]
            sigma[(ga, gc)] = blk
        ha = rows_last if ga == part.last else b
        diag[ga * b:ga * b + ha] = np.diag(red.sigma)[a * b:a * b + ha]
    return sigma, diag


def dist_allreduce(dist, device=None):
    """all-reduce (sum) of the reduced system and the interior logdet over the
    process group: NCCL on the GPUs' own tensors (device = "cuda:k"), gloo on
    CPU tensors.  Returns the `allreduce(G, x) -> (G, x)` hook of `run`."""
    import torch

    def allreduce(G, x):
        t = torch.from_numpy(np.ascontiguousarray(G))
        s = torch.tensor([x], dtype=torch.float64)
        if device is not None:
            t = t.to(device)
            s = s.to(device)
        dist.all_reduce(t)
        dist.all_reduce(s)
        return t.cpu().numpy(), float(s.item())

    return allreduce


def selected_inverse_partitioned(matrix, parts: int, rank: int = 0, world: int = 1, allreduce=None, device: int = 0,
                                 engine=None):
    """Partitioned selected inversion of one band+arrow matrix (marginal
    variances and Sigma on the matrix's own pattern, logdet).  `world == 1`
    runs every part in this process (the collective is a local sum);
    otherwise part p runs on rank p (parts == world) and `allreduce` is
    dist_allreduce(...).  Returns (PartResults of this rank, ReducedResult,
    logdet, partition, TileMap)."""
    ti, tj, pay = matrix.tiles()
    A = TileMap(matrix.n, matrix.tile_size, ti, tj, pay)
    bw, na = band_of(ti, tj, A.N)
    part = BandArrowPartition(A.N, bw, parts, na)
    if world == 1:
        mine, allreduce = list(range(parts)), (lambda G, x: (G, x))
    else:
        if parts != world:
            raise ValueError("one part per rank")
        mine = [rank]
    eng = engine or DeviceEngine(device)
    res, red, ld = run(A, part, mine, eng, allreduce)
    return res, red, ld, part, A
