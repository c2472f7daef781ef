"""The device task plans, executed on the CPU by tests/plan_sim.py (numpy block
products, in-order two-queue claiming), reproduce the oracle: this checks the
dataflow decomposition, operand addressing, dependency counters and queue
order without a GPU, and that the order is deadlock-free with one worker per
queue."""
import os

import numpy as np
import pytest

from conftest import normwise
from plan_sim import run_plans


CASES = [
    (700, 90, 12, 1.0, 5, 64, "pattern"),
    (300, 40, 7, 1.0, 3, 32, "all"),
    (520, 150, 20, 1.0, 11, 128, "pattern"),
    (260, 60, 9, 0.4, 2, 128, "diagonal"),
    (300, 40, 7, 1.0, 3, 32, [(299, 0), (150, 3), (5, 5), (200, 100)]),
    (400, 0, 30, 1.0, 4, 64, "pattern"),       # no band: diagonal + arrow only
    (1100, 300, 40, 1.0, 9, 256, "pattern"),   # bp = 256: 4x4 blocks per tile
    (1000, 0, 100, 1.0, 4, 100, "pattern"),    # arrow only, t >= b: first off-diagonal tile is not j + 1
]


@pytest.mark.parametrize("case", CASES, ids=[str(c[:6]) for c in CASES])
def test_plan_simulation_matches_oracle(tib, orc, case):
    n, w, t, d, seed, b, sel = case
    m = tib.generate(n, w, t, d, seed=seed, tile_size=b)
    fpat, closure, sig, logdet, bad, var = run_plans(tib, m, sel)
    ref = orc.selected_inverse_generated(n, w, t, d, seed, b, sel)
    assert closure == ref["tiles"]
    assert normwise(sig, ref["payload"]) <= 1e-12
    assert abs(logdet - ref["logdet"]) <= 1e-12 * abs(ref["logdet"])
    assert bad == np.iinfo(np.int64).max
    if ref["diag"] is not None:
        assert normwise(var, ref["diag"]) <= 1e-12


def test_plan_simulation_reports_not_spd(tib):
    a = np.eye(6)
    a[4, 4] = -1.0  # test_cholesky.cpp:161-182: pivot 4, tile (2, 2) at b = 2
    m = tib.from_dense(a, tile_size=2)
    *_, bad, _ = run_plans(tib, m, "pattern")
    assert bad == 4


def test_plans_are_topological_for_every_selection(tib):
    # building a plan runs validate_dataflow (plan.cpp), which throws on any
    # dependency not produced earlier in emission order
    m = tib.generate(3000, 400, 60, 0.3, seed=1, tile_size=100)
    for sel in ("pattern", "diagonal", "all", [(2999, 5), (10, 10)]):
        for which in (0, 1):
            p = tib.plan_export(m, sel, which, crit_workers=8)
            assert len(p["tasks"]) > 0 and p["q0"] > 0


def gapped_arrow(n=900, blocks=(0, 300, 520, 760), t=70, seed=3):
    """Block-diagonal SPD blocks plus a dense arrow: a tile pattern with gaps
    below the diagonal (first off-diagonal tile of a column != j + 1)."""
    rng = np.random.default_rng(seed)
    a = np.zeros((n, n))
    edges = list(blocks) + [n - t]
    for lo, hi in zip(edges[:-1], edges[1:]):
        m = rng.uniform(-1, 1, (hi - lo, hi - lo))
        a[lo:hi, lo:hi] = (m + m.T) / 2
    a[n - t:, :] = rng.uniform(-1, 1, (t, n))
    a[:, n - t:] = a[n - t:, :].T
    a = (a + a.T) / 2
    a[np.diag_indices(n)] = np.abs(a).sum(1) + 1.0
    return a


def test_plan_simulation_gapped_pattern(tib):
    a = gapped_arrow()
    m = tib.from_dense(a, tile_size=128)
    _, closure, sig, logdet, _, var = run_plans(tib, m, "pattern")
    inv = np.linalg.inv(a)
    assert abs(logdet - np.linalg.slogdet(a)[1]) <= 1e-12 * abs(logdet)
    assert normwise(var, np.diag(inv)) <= 1e-12


@pytest.mark.parametrize("seed", [0, 1, 2])
@pytest.mark.parametrize("case", [
    (700, 90, 12, 1.0, 5, 64, "pattern"),
    (520, 150, 20, 1.0, 11, 128, "pattern"),
    (1000, 0, 100, 1.0, 4, 100, "pattern"),
    (1100, 300, 40, 1.0, 9, 256, "pattern"),
], ids=lambda c: str(c[:6]) if isinstance(c, tuple) else str(c))
def test_plan_simulation_random_order(tib, orc, case, seed):
    """Any ready task may run at any time on the GPU: a random ready order
    must give the same result (catches dependencies missing from the plan)."""
    n, w, t, d, s, b, sel = case
    m = tib.generate(n, w, t, d, seed=s, tile_size=b)
    _, closure, sig, logdet, _, var = run_plans(tib, m, sel, order=seed)
    ref = orc.selected_inverse_generated(n, w, t, d, s, b, sel)
    assert normwise(sig, ref["payload"]) <= 1e-12
    assert abs(logdet - ref["logdet"]) <= 1e-12 * abs(ref["logdet"])


@pytest.mark.parametrize("seed", [0, 1])
def test_plan_simulation_gapped_random(tib, seed):
    a = gapped_arrow()
    m = tib.from_dense(a, tile_size=128)
    _, closure, sig, logdet, _, var = run_plans(tib, m, "pattern", order=seed)
    assert normwise(var, np.diag(np.linalg.inv(a))) <= 1e-12


TWO_CHAIN = [
    (3000, 200, 30, 1.0, 3, 64),    # band 4 tiles + arrow
    (4096, 300, 0, 1.0, 8, 128),    # no arrow, n a multiple of b: the last band tile moves too
    (5000, 500, 60, 1.0, 2, 256),   # bp = 256, arrow straddling two tile rows
]


@pytest.mark.parametrize("case", TWO_CHAIN, ids=[str(c) for c in TWO_CHAIN])
@pytest.mark.parametrize("order", [None, 1])
def test_plan_simulation_two_chains(tib, orc, case, order):
    """The two-chain elimination order (interior 1 reversed, separator, arrow):
    the permuted matrix has the original's tile count (no fill), its split
    factor plan (two chains, one scratch ring each) reproduces the oracle on
    the permuted matrix, and Sigma's diagonal and the logdet equal the
    natural-order oracle's to rounding."""
    n, w, t, d, seed, b = case
    m = tib.generate(n, w, t, d, seed=seed, tile_size=b)
    perm, split = tib.two_chain_order(m)
    assert split > 0
    mp = tib.two_chain_permuted(m)
    assert mp.stored_tiles == len(tib.factor_pattern(m))
    fpat, closure, sig, logdet, bad, var = run_plans(tib, mp, "pattern", order=order, split=split)
    ti, tj, pay = mp.tiles()
    ref = orc.selected_inverse(n, b, mp.n_tiles, list(zip(ti.tolist(), tj.tolist())), pay, "pattern")
    assert closure == ref["tiles"]
    assert normwise(sig, ref["payload"]) <= 1e-12
    assert bad == np.iinfo(np.int64).max
    nat = orc.selected_inverse_generated(n, w, t, d, seed, b, "pattern")
    assert abs(logdet - nat["logdet"]) <= 1e-12 * abs(nat["logdet"])
    # diag of the permuted matrix, rows mapped back tile by tile
    N = m.n_tiles
    back = np.zeros(n)
    for k in range(N):
        rows = min(b, n - perm[k] * b)
        back[perm[k] * b: perm[k] * b + rows] = var[k * b: k * b + rows]
    assert normwise(back, nat["diag"]) <= 1e-12


@pytest.mark.parametrize("case", CASES[:3] + CASES[5:], ids=[str(c[:6]) for c in CASES[:3] + CASES[5:]])
@pytest.mark.parametrize("order", [None, 3])
def test_plan_simulation_batch_plans(tib, orc, case, order):
    """The plans of a batched launch (more than 4 matrices): plain leaf tasks
    instead of the chain task, phase-2 late terms three to a part."""
    n, w, t, d, seed, b, sel = case
    if sel != "pattern":
        return
    m = tib.generate(n, w, t, d, seed=seed, tile_size=b)
    fpat, closure, sig, logdet, bad, var = run_plans(tib, m, sel, order=order, batch=64)
    ref = orc.selected_inverse_generated(n, w, t, d, seed, b, sel)
    assert closure == ref["tiles"]
    assert normwise(sig, ref["payload"]) <= 1e-12
    assert abs(logdet - ref["logdet"]) <= 1e-12 * abs(ref["logdet"])


@pytest.mark.parametrize("group", [2, 3, 5])
@pytest.mark.parametrize("case", [
    (700, 90, 12, 1.0, 5, 64, "pattern"),      # band 2 tiles: groups cut by the tile's next use
    (1100, 300, 40, 1.0, 9, 64, "pattern"),    # band 5 tiles: full groups
    (1000, 0, 100, 1.0, 4, 100, "pattern"),    # arrow only
], ids=lambda c: str(c[:6]) if isinstance(c, tuple) else str(c))
@pytest.mark.parametrize("order", [None, 1])
def test_plan_simulation_grouped_updates(tib, orc, monkeypatch, case, group, order):
    """Bulk update terms grouped `group` to a factor task (multi-segment GEMMs,
    signals repeated per term) in the chain plan, a batch plan and a random
    ready order: Sigma and logdet still equal the oracle's."""
    monkeypatch.setenv("TIB_UPD_GROUP", str(group))
    n, w, t, d, seed, b, sel = case
    m = tib.generate(n, w, t, d, seed=seed, tile_size=b)
    ref = orc.selected_inverse_generated(n, w, t, d, seed, b, sel)
    for batch in (1, 64):
        _, closure, sig, logdet, _, var = run_plans(tib, m, sel, order=order, batch=batch)
        assert closure == ref["tiles"]
        assert normwise(sig, ref["payload"]) <= 1e-12
        assert abs(logdet - ref["logdet"]) <= 1e-12 * abs(ref["logdet"])
