"""Pins the CPU oracle (oracle/tileinv_oracle.c + oracle/oracle.py) against the
reference: its known-answer tests, the committed golden fixtures made by the
reference itself, and -- where oracle/_ref is built -- live reference runs."""
import json
import os

import numpy as np
import pytest

from conftest import GOLDEN, elementwise, normwise


def oracle_entries(orc, n, w, t, d, seed, b, sel):
    res = orc.selected_inverse_generated(n, w, t, d, seed, b, sel)
    N = (n + b - 1) // b
    idx = {tile: k for k, tile in enumerate(res["tiles"])}
    order = orc.entries_order(n, b, N, res["tiles"], res["requested"], sel)
    vals = []
    for r, c in order:
        rr, cc = max(r, c), min(r, c)
        vals.append(res["payload"][idx[(rr // b, cc // b)], rr % b, cc % b])
    return np.array(order, dtype=np.int64).reshape(-1, 2), np.array(vals)


def test_oracle_known_answers(orc):
    # test_smoke.py:19-25 / test_selinv.cpp:381-392: [[4,2],[2,5]] -> [[5/16,-1/8],[-1/8,1/4]]
    N, tiles, pay = orc.tiles_from_dense(np.array([[4.0, 2.0], [2.0, 5.0]]), 32)
    res = orc.selected_inverse(2, 32, N, tiles, pay, "all")
    s = res["payload"][0]
    assert s[0, 0] == 0.3125 and s[1, 0] == -0.125 and s[1, 1] == 0.25
    # test_kernels.cpp:72-81 potrf [[4]] -> [[2]]; trtri [[2]] -> [[0.5]] (phase-1 U)
    N, tiles, pay = orc.tiles_from_dense(np.array([[4.0]]), 1)
    res = orc.selected_inverse(1, 1, N, tiles, pay, "all")
    assert res["factor"][0, 0, 0] == 2.0 and res["phase1"][0, 0, 0] == 0.5 and res["payload"][0, 0, 0] == 0.25
    # test_selinv.cpp:279-295: diagonal inverse 0.25 / 0.5 / 0.1 / 2.0
    N, tiles, pay = orc.tiles_from_dense(np.diag([4.0, 2.0, 10.0, 0.5]), 2)
    res = orc.selected_inverse(4, 2, N, tiles, pay, "diagonal")
    assert np.allclose(res["diag"], [0.25, 0.5, 0.1, 2.0], rtol=1e-15)
    # test_cholesky.cpp:161-182: NotSpd at global pivot 4 (tile (2, 2)) for b = 2
    d = np.eye(6)
    d[4, 4] = -1.0
    N, tiles, pay = orc.tiles_from_dense(d, 2)
    assert orc.selected_inverse(6, 2, N, tiles, pay, "pattern")["not_spd_pivot"] == 4


def test_oracle_matches_reference_goldens(orc):
    cases = json.load(open(os.path.join(GOLDEN, "symbolic.json")))
    arrays = np.load(os.path.join(GOLDEN, "cases.npz"))
    for key, case in cases.items():
        n, w, t, d, seed, b, sel = case["args"]
        if not isinstance(sel, str):
            sel = [tuple(p) for p in sel]
        want = arrays[key]
        order, vals = oracle_entries(orc, n, w, t, d, seed, b, sel)
        assert np.array_equal(order, want[:, :2].astype(np.int64)), key
        assert normwise(vals, want[:, 2]) <= 1e-13, key
        # symbolic half of the oracle vs the reference's own planner
        N = (n + b - 1) // b
        _, tiles, _ = orc.generate(n, w, t, d, seed, b)
        filled = orc.symbolic_fill(N, tiles)
        assert filled == [tuple(x) for x in case["factor"]], key
        req = orc.select_tiles(n, b, N, filled, sel)
        closure, work = orc.symbolic_inversion(N, req, filled)
        assert closure == [tuple(x) for x in case["closure"]], key
        assert [(c, int(dg), list(rows)) for c, dg, rows in work] == [(c, dg, rows) for c, dg, rows in case["columns"]]


def test_oracle_small_config_goldens(orc):
    """SURVEY.md 6.2 small config: logdet / trace / diag(Sigma) of the reference."""
    g = np.load(os.path.join(GOLDEN, "small.npz"))
    res = orc.selected_inverse_generated(10000, 200, 50, 1.0, 42, 128, "pattern")
    assert abs(res["logdet"] - float(g["logdet"])) / abs(float(g["logdet"])) <= 1e-13
    assert elementwise(res["diag"], g["diag"]) <= 1e-12
    assert abs(res["logdet"] - 5.423829124603e04) / 5.423829124603e04 < 1e-12
    assert abs(res["diag"].sum() - 4.475492240168e01) < 1e-10


def test_oracle_generator_bit_exact_vs_reference(orc, ref):
    for (n, w, t, d, seed, b) in [(24, 5, 2, 0.8, 7, 4), (300, 40, 7, 1.0, 3, 32), (129, 20, 9, 0.4, 5, 16)]:
        N, tiles, pay = orc.generate(n, w, t, d, seed, b)
        dense = np.zeros((N * b, N * b))
        for (i, j), tile in zip(tiles, pay):
            dense[i * b:(i + 1) * b, j * b:(j + 1) * b] = tile
        dense = np.tril(dense)[:n, :n]
        dense = dense + np.tril(dense, -1).T
        assert np.array_equal(dense, ref.generate(n, w, t, d, seed=seed, tile_size=b).to_dense())


@pytest.mark.parametrize("sel", ["all", "diagonal", "pattern"])
def test_oracle_vs_live_reference(orc, ref, sel):
    n, w, t, d, seed, b = 130, 20, 6, 0.7, 19, 16
    res = ref.selected_inverse(ref.generate(n, w, t, d, seed=seed, tile_size=b), sel)
    want = np.array(res.entries()).reshape(-1, 3)
    order, vals = oracle_entries(orc, n, w, t, d, seed, b, sel)
    assert np.array_equal(order, want[:, :2].astype(np.int64))
    assert normwise(vals, want[:, 2]) <= 1e-13
