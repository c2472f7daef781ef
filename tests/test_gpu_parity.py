"""GPU parity: the sm_100a path through the C ABI against the reference's
known answers, the golden fixtures made by the reference, and the CPU oracle.

Gate: Sigma tiles normwise <= 1e-10, diag(Sigma)
elementwise <= 1e-10, logdet relative <= 1e-10, tile pattern identical.
Elementwise max_rel_error over all Sigma entries is information only (two
valid CPU tilings already differ by 3.7e-10)."""
import json
import os

import numpy as np
import pytest

from conftest import GOLDEN, elementwise, normwise

pytestmark = pytest.mark.gpu
TOL = 1e-10


def entries_array(res):
    r, c, v = res.entries_arrays()
    return np.stack([r, c], 1), v


def test_known_answers(tib):
    # test_smoke.py:19-25, test_selinv.cpp:381-392
    got = {(r, c): v for r, c, v in tib.selected_inverse(tib.from_dense(np.array([[4.0, 2.0], [2.0, 5.0]])),
                                                          "all").entries()}
    assert got[(0, 0)] == 0.3125 and got[(1, 0)] == -0.125 and got[(1, 1)] == 0.25
    # test_smoke.py:11-16
    ent = tib.selected_inverse(tib.from_dense(np.eye(5), tile_size=2), "diagonal").entries()
    assert [(r, c) for r, c, _ in ent] == [(i, i) for i in range(5)] and all(v == 1.0 for *_, v in ent)
    # test_selinv.cpp:279-295
    d = tib.selected_inverse(tib.from_dense(np.diag([4.0, 2.0, 10.0, 0.5]), tile_size=2), "diagonal").diagonal()
    assert np.allclose(d, [0.25, 0.5, 0.1, 2.0], rtol=1e-15, atol=0)


def test_not_spd(tib):
    # test_smoke.py:75-78
    with pytest.raises(tib.NotSpdError):
        tib.factorize(tib.from_dense(np.array([[1.0, 2.0], [2.0, 1.0]])))
    # test_cholesky.cpp:161-182: global pivot 4, tile (2, 2)
    a = np.eye(6)
    a[4, 4] = -1.0
    with pytest.raises(tib.NotSpdError) as e:
        tib.factorize(tib.from_dense(a, tile_size=2))
    assert (e.value.pivot, e.value.tile_i, e.value.tile_j) == (4, 2, 2)
    with pytest.raises(tib.NotSpdError):
        tib.selected_inverse(tib.from_dense(a, tile_size=2), "diagonal")


def test_reference_golden_cases(tib):
    cases = json.load(open(os.path.join(GOLDEN, "symbolic.json")))
    arrays = np.load(os.path.join(GOLDEN, "cases.npz"))
    for key, case in cases.items():
        n, w, t, d, seed, b, sel = case["args"]
        if not isinstance(sel, str):
            sel = [tuple(p) for p in sel]
        res = tib.selected_inverse(tib.generate(n, w, t, d, seed=seed, tile_size=b), sel)
        want = arrays[key]
        idx, vals = entries_array(res)
        assert np.array_equal(idx, want[:, :2].astype(np.int64)), key
        assert normwise(vals, want[:, 2]) <= TOL, key
        assert res.closure_tiles == len(case["closure"])


@pytest.mark.parametrize("case", [
    (24, 5, 2, 0.8, 7, 4, "all"),
    (37, 6, 3, 1.0, 1, 1, "all"),            # b = 1
    (101, 9, 4, 0.9, 2, 3, "pattern"),       # b = 3
    (300, 40, 7, 1.0, 3, 32, "all"),
    (700, 90, 12, 1.0, 5, 64, "pattern"),
    (1000, 0, 25, 1.0, 6, 100, "pattern"),   # no band, b not a multiple of 64
    (1500, 300, 0, 1.0, 9, 128, "pattern"),  # no arrow
    (2000, 150, 12, 0.2, 4, 256, "pattern"),
    (2600, 400, 30, 1.0, 7, 120, "diagonal"),
    (3000, 700, 50, 1.0, 1, 512, "pattern"),
    (1200, 200, 20, 1.0, 8, 96, [(1199, 0), (600, 3), (5, 5), (700, 650), (5, 5)]),
])
def test_parity_vs_oracle(tib, orc, case):
    n, w, t, d, seed, b, sel = case
    res = tib.selected_inverse(tib.generate(n, w, t, d, seed=seed, tile_size=b), sel)
    ref = orc.selected_inverse_generated(n, w, t, d, seed, b, sel)
    ti, tj, pay = res.tiles()
    assert list(zip(ti.tolist(), tj.tolist())) == ref["tiles"]
    assert normwise(pay, ref["payload"]) <= TOL
    assert abs(res.logdet() - ref["logdet"]) <= TOL * abs(ref["logdet"])
    if ref["diag"] is not None:
        assert elementwise(res.diagonal(), ref["diag"]) <= TOL
    # diagonal tiles exactly symmetric (selinv.cpp:319-321)
    for k in range(len(ti)):
        if ti[k] == tj[k]:
            assert np.array_equal(pay[k], pay[k].T)


def test_small_config_vs_reference(tib, orc):
    """SURVEY small config (CPU-runnable reference case): diag, logdet vs the
    reference's own run, Sigma tiles vs the oracle."""
    g = np.load(os.path.join(GOLDEN, "small.npz"))
    m = tib.generate(10000, 200, 50, 1.0, seed=42, tile_size=128)
    res = tib.selected_inverse(m, "pattern")
    assert elementwise(res.diagonal(), g["diag"]) <= TOL
    assert abs(res.logdet() - float(g["logdet"])) <= TOL * abs(float(g["logdet"]))
    ref = orc.selected_inverse_generated(10000, 200, 50, 1.0, 42, 128, "pattern")
    ti, tj, pay = res.tiles()
    assert list(zip(ti.tolist(), tj.tolist())) == ref["tiles"]
    assert normwise(pay, ref["payload"]) <= TOL
    # per tile column too
    scale = np.abs(ref["payload"]).max()
    for j in np.unique(tj):
        sl = tj == j
        assert np.abs(pay[sl] - ref["payload"][sl]).max() / scale <= TOL
    info = elementwise(pay, ref["payload"], floor=1e-30)
    print(f"elementwise max_rel_error (information only): {info:.3e}")


def test_factor_path_and_determinism(tib, orc):
    n, w, t, d, seed, b = 3000, 300, 40, 1.0, 17, 128
    m = tib.generate(n, w, t, d, seed=seed, tile_size=b)
    f = tib.factorize(m, workers=2)
    ref = orc.selected_inverse_generated(n, w, t, d, seed, b, "pattern")
    _, _, L = f.tiles(1)
    assert normwise(L, ref["factor"]) <= TOL
    _, _, P1 = f.tiles(2)
    assert normwise(P1, ref["phase1"]) <= TOL
    assert abs(f.logdet() - ref["logdet"]) <= TOL * abs(ref["logdet"])
    via = tib.selected_inverse_of_factor(f, "pattern")
    direct = tib.selected_inverse(m, "pattern")
    again = tib.selected_inverse(m, "pattern")
    # fixed accumulation order, no atomics on data: bitwise reproducible
    assert direct.checksum == again.checksum == via.checksum
    assert f.checksum == tib.factorize(m).checksum
    # one factor serves several requests (module.cpp:208-215)
    diag = tib.selected_inverse_of_factor(f, "diagonal")
    assert elementwise(diag.diagonal(), ref["diag"]) <= TOL


@pytest.mark.parametrize("count", [3, 6, 80])  # 6 > TIB_DEDICATE_MAX_BATCH: chains share their SMs;
# 80 > the reserved critical workers: every chain still runs on its own worker
def test_batch_matches_single(tib, count):
    b = 256 if count > 6 else 128
    ms = [tib.generate(5000, 500, 50, 1.0, seed=1000 + k, tile_size=b) for k in range(count)]
    logdet, diag = tib.selected_inverse_batch(ms)
    for k in (range(count) if count <= 6 else (0, 1, count - 2, count - 1)):
        res = tib.selected_inverse(ms[k], "pattern")
        assert logdet[k] == res.logdet()
        assert np.array_equal(diag[k], res.diagonal())


def test_streamed_upload_is_bitwise_identical(tib, monkeypatch):
    """The public path streams A up column by column under the factor sweep
    (tasks poll per-column upload counters); the result must not depend on it."""
    m = tib.generate(6000, 700, 60, 1.0, seed=23, tile_size=256)
    streamed = tib.selected_inverse(m, "pattern")
    monkeypatch.setenv("TIB_STREAM_UPLOAD", "0")
    upfront = tib.selected_inverse(m, "pattern")
    assert streamed.checksum == upfront.checksum
    assert streamed.logdet() == upfront.logdet()


@pytest.mark.parametrize("b", [256, 512])
def test_eight_warp_chain_is_bitwise_identical(tib, monkeypatch, b):
    """The experimental eight-warp chain (TIB_CHAIN8=1: a helper worker stores
    each leaf, raises the chain's signals and forms the lookahead products)
    performs the same operations in the same order as the default chain."""
    m = tib.generate(9000, 900, 60, 1.0, seed=29, tile_size=b)
    ref = tib.selected_inverse(m, "pattern")
    monkeypatch.setenv("TIB_CHAIN8", "1")
    alt = tib.selected_inverse(m, "pattern")
    assert alt.checksum == ref.checksum
    assert alt.logdet() == ref.logdet()


@pytest.mark.parametrize("cfg", [
    ("medium", 100000, 1000, 100, 256, 6.955199016515e05, 9.580956859578e01),
    ("large", 200000, 2000, 200, 512, 1.529607821236e06, 9.582054347524e01),
])
def test_full_size_goldens(tib, cfg):
    """Full BASELINE sizes (size-independent properties): logdet and
    trace(Sigma) against the reference's values (SURVEY.md 6.2, 13 significant
    digits) and positive marginal variances."""
    _, n, w, t, b, ld_ref, tr_ref = cfg
    m = tib.generate(n, w, t, 1.0, seed=42, tile_size=b)
    res = tib.selected_inverse(m, "pattern")
    assert abs(res.logdet() - ld_ref) / ld_ref < 5e-13
    d = res.diagonal()
    assert abs(d.sum() - tr_ref) / tr_ref < 5e-12
    assert np.all(d > 0)
