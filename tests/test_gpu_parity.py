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


def test_factor_path_and_determinism(tib, orc, monkeypatch):
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
    monkeypatch.setenv("TIB_SPLIT_STREAMED", "1")  # the two-chain order, streamed
    monkeypatch.setenv("TIB_SPLIT_AGENTS", "1")
    direct = tib.selected_inverse(m, "pattern")
    again = tib.selected_inverse(m, "pattern")
    # fixed accumulation order, no atomics on data: bitwise reproducible
    assert direct.checksum == again.checksum
    assert normwise(direct.tiles()[2], via.tiles()[2]) <= 1e-13
    # the natural elimination order is the factor's: the same bits
    monkeypatch.setenv("TIB_SPLIT", "0")
    assert tib.selected_inverse(m, "pattern").checksum == via.checksum
    assert f.checksum == tib.factorize(m).checksum
    # one factor serves several requests (module.cpp:208-215)
    diag = tib.selected_inverse_of_factor(f, "diagonal")
    assert elementwise(diag.diagonal(), ref["diag"]) <= TOL


@pytest.mark.parametrize("count", [3, 6, 80])  # 6 > TIB_DEDICATE_MAX_BATCH: chains share their SMs;
# 80 > the reserved critical workers: every chain still runs on its own worker
def test_batch_matches_single(tib, count, monkeypatch):
    b = 256 if count > 6 else 128
    ms = [tib.generate(5000, 500, 50, 1.0, seed=1000 + k, tile_size=b) for k in range(count)]
    # a batch of more than 4 runs plain leaf tasks and groups phase 2's late
    # terms: the same values to rounding
    logdet, diag = tib.selected_inverse_batch(ms)
    monkeypatch.setenv("TIB_SPLIT", "0")  # single calls in the batch's (natural) elimination order
    for k in (0, count - 1):
        res = tib.selected_inverse(ms[k], "pattern")
        assert abs(logdet[k] - res.logdet()) <= 1e-13 * abs(res.logdet())
        assert elementwise(diag[k], res.diagonal()) <= 1e-12
    # with the single call's task structure, the same bits
    monkeypatch.setenv("TIB_BATCH_CHAIN", "1")
    monkeypatch.setenv("TIB_P2_GROUP", "1")
    logdet, diag = tib.selected_inverse_batch(ms)
    for k in (range(count) if count <= 6 else (0, 1, count - 2, count - 1)):
        res = tib.selected_inverse(ms[k], "pattern")
        assert logdet[k] == res.logdet()
        assert np.array_equal(diag[k], res.diagonal())


@pytest.mark.parametrize("split", ["0", "1"])
def test_streamed_upload_is_bitwise_identical(tib, monkeypatch, split):
    """The public path streams A up column by column under the factor sweep
    (tasks poll per-column upload counters); the result must not depend on it,
    in either elimination order."""
    monkeypatch.setenv("TIB_SPLIT", split)
    monkeypatch.setenv("TIB_SPLIT_STREAMED", split)
    monkeypatch.setenv("TIB_SPLIT_AGENTS", "1")
    m = tib.generate(6000, 700, 60, 1.0, seed=23, tile_size=256)
    streamed = tib.selected_inverse(m, "pattern")
    monkeypatch.setenv("TIB_STREAM_UPLOAD", "0")
    upfront = tib.selected_inverse(m, "pattern")
    assert streamed.checksum == upfront.checksum
    assert streamed.logdet() == upfront.logdet()


@pytest.mark.parametrize("how", ["streamed", "upfront", "device"])
def test_two_chain_order_matches_natural(tib, orc, monkeypatch, how):
    """Single-matrix calls run in the two-chain elimination order (interior 1
    reversed, separator, arrow) with Sigma un-permuted on the
    device: Sigma, the marginal variances and the logdet equal the natural
    order's (and the oracle's) to rounding, for every upload path."""
    n, w, t, seed, b = 9000, 600, 70, 31, 128
    m = tib.generate(n, w, t, 1.0, seed=seed, tile_size=b, device=0 if how == "device" else None)
    assert tib.two_chain_order(m)[1] > 0
    if how == "upfront":
        monkeypatch.setenv("TIB_STREAM_UPLOAD", "0")
    if how == "streamed":  # host inputs stream in the natural order unless asked
        monkeypatch.setenv("TIB_SPLIT_STREAMED", "1")
        monkeypatch.setenv("TIB_SPLIT_AGENTS", "1")
    got = tib.selected_inverse(m, "pattern")
    monkeypatch.setenv("TIB_SPLIT", "0")
    nat = tib.selected_inverse(m, "pattern")
    assert got.checksum != nat.checksum  # (the two orders round differently: the split path ran)
    ti, tj, pay = got.tiles()
    ti2, tj2, pay2 = nat.tiles()
    assert np.array_equal(ti, ti2) and np.array_equal(tj, tj2)
    assert normwise(pay, pay2) <= 1e-13
    assert elementwise(got.diagonal(), nat.diagonal()) <= 1e-12
    assert abs(got.logdet() - nat.logdet()) <= 1e-13 * abs(nat.logdet())
    ref = orc.selected_inverse_generated(n, w, t, 1.0, seed, b, "pattern")
    assert normwise(pay, ref["payload"]) <= TOL
    assert elementwise(got.diagonal(), ref["diag"]) <= TOL
    # exactly symmetric diagonal tiles survive the un-permutation
    for k in np.nonzero(ti == tj)[0][:8]:
        assert np.array_equal(pay[k], pay[k].T)
    # entries in the reference's order, like the natural call
    r1, c1, v1 = got.entries_arrays()
    r2, c2, v2 = nat.entries_arrays()
    assert np.array_equal(r1, r2) and np.array_equal(c1, c2)
    assert normwise(v1, v2) <= 1e-13


def test_two_chain_not_spd_reports_the_natural_pivot(tib):
    """A NotSpd in the permuted elimination is re-run in the natural order, so
    the error carries the reference's first non-positive pivot."""
    m = tib.generate(6000, 500, 40, 1.0, seed=3, tile_size=128)
    ti, tj, pay = m.tiles()
    pay = pay.copy()
    k = int(np.nonzero((ti == tj) & (ti == 30))[0][0])
    pay[k][5, 5] = -1.0
    bad = tib.from_tiles(m.n, 128, ti, tj, pay)
    assert tib.two_chain_order(bad)[1] > 0
    with pytest.raises(tib.NotSpdError) as e:
        tib.selected_inverse(bad, "pattern")
    with pytest.raises(tib.NotSpdError) as e2:
        tib.factorize(bad)
    assert (e.value.pivot, e.value.tile_i) == (e2.value.pivot, e2.value.tile_i)


def test_diagonal_tiles_lower_triangle_only(tib, monkeypatch):
    """Diagonal tiles of A are significant in their lower triangle only (the
    reference's potrf reads the lower part, kernels.cpp:48-69): garbage in the
    strict upper part changes nothing, streamed upload or not."""
    monkeypatch.setenv("TIB_SPLIT", "0")  # the same elimination order for both uploads
    m = tib.generate(6000, 700, 60, 1.0, seed=29, tile_size=128)
    ti, tj, pay = m.tiles()
    ref = tib.selected_inverse(m, "pattern")
    junk = pay.copy()
    rng = np.random.default_rng(5)
    up = np.triu(np.ones((128, 128), bool), 1)
    for k in np.nonzero(ti == tj)[0]:
        junk[k][up] = rng.uniform(-1e3, 1e3, up.sum())
    mj = tib.from_tiles(m.n, 128, ti, tj, junk)
    for stream in ("1", "0"):
        monkeypatch.setenv("TIB_STREAM_UPLOAD", stream)
        got = tib.selected_inverse(mj, "pattern")
        assert got.checksum == ref.checksum, stream
        assert got.logdet() == ref.logdet()


def test_gapped_patterns_vs_dense(tib):
    """Tile patterns whose first off-diagonal tile is not j + 1: the chain's
    boundary step must write the next diagonal block back."""
    from test_plan_sim import gapped_arrow

    for a, b in ((gapped_arrow(), 128), (gapped_arrow(1400, (0, 256, 700, 1000), 150, 5), 256)):
        res = tib.selected_inverse(tib.from_dense(a, tile_size=b), "pattern")
        inv = np.linalg.inv(a)
        assert elementwise(res.diagonal(), np.diag(inv)) <= TOL
        assert abs(res.logdet() - np.linalg.slogdet(a)[1]) <= TOL * abs(res.logdet())
        ti, tj, pay = res.tiles()
        n = a.shape[0]
        for k in range(len(ti)):
            r0, c0 = ti[k] * b, tj[k] * b
            blk = inv[r0:r0 + b, c0:c0 + b]
            assert np.abs(pay[k][:blk.shape[0], :blk.shape[1]] - blk).max() <= TOL * np.abs(inv).max()


@pytest.mark.parametrize("case", [
    (1000, 0, 100, 1.0, 4, 100, "pattern"),   # arrow only, t >= b, bp = 128
    (3000, 0, 600, 1.0, 6, 512, "pattern"),   # arrow only over two tile rows
    (4000, 0, 300, 1.0, 2, 256, "diagonal"),
])
def test_arrow_only_vs_oracle(tib, orc, case):
    n, w, t, d, seed, b, sel = case
    res = tib.selected_inverse(tib.generate(n, w, t, d, seed=seed, tile_size=b), sel)
    ref = orc.selected_inverse_generated(n, w, t, d, seed, b, sel)
    _, _, pay = res.tiles()
    assert normwise(pay, ref["payload"]) <= TOL
    assert elementwise(res.diagonal(), ref["diag"]) <= TOL
    assert abs(res.logdet() - ref["logdet"]) <= TOL * abs(ref["logdet"])


def test_batch_larger_than_one_launch(tib, monkeypatch):
    """More matrices than CTAs (static chain assignment) and more than the
    old 7-bit item packing allowed: the engine runs the batch in launches of
    at most one chain per CTA."""
    monkeypatch.setenv("TIB_SPLIT", "0")  # single calls in the batch's order, tasks and grouping
    monkeypatch.setenv("TIB_P2_GROUP", "1")
    monkeypatch.setenv("TIB_BATCH_CHAIN", "1")
    ms = [tib.generate(300, 40, 7, 1.0, seed=500 + k, tile_size=64) for k in range(300)]
    logdet, diag = tib.selected_inverse_batch(ms)
    for k in (0, 127, 128, 147, 148, 299):
        res = tib.selected_inverse(ms[k], "pattern")
        assert logdet[k] == res.logdet()
        assert np.array_equal(diag[k], res.diagonal())


def test_watchdog_turns_a_stall_into_an_error(tib, monkeypatch):
    """A sweep that can never finish (test hook: one task never becomes
    ready) ends with TileinvError from the executor's watchdog instead of
    hanging the process."""
    monkeypatch.setenv("TIB_TEST_STALL", "1")
    monkeypatch.setenv("TIB_WATCHDOG_S", "2")
    m = tib.generate(1777, 111, 13, 1.0, seed=3, tile_size=96)  # a pattern no other test plans
    with pytest.raises(tib.TileinvError, match="watchdog"):
        tib.selected_inverse(m, "pattern")
    monkeypatch.delenv("TIB_TEST_STALL")
    # the device stays usable
    res = tib.selected_inverse(tib.generate(700, 90, 12, 1.0, seed=5, tile_size=64), "pattern")
    assert np.all(res.diagonal() > 0)


@pytest.mark.parametrize("group", ["1", "2", "16"])
def test_grouped_updates_match_oracle(tib, orc, monkeypatch, group):
    """Bulk update terms grouped 1 / 2 / 16 to a factor task (TIB_UPD_GROUP;
    default 4) in the two-chain order and in a launch of 33 matrices (leaf
    plans): Sigma, the marginal variances and the logdet match the oracle."""
    monkeypatch.setenv("TIB_UPD_GROUP", group)
    n, w, t, b = 6000, 700, 60, 128
    ref = orc.selected_inverse_generated(n, w, t, 1.0, 7, b, "pattern")
    m = tib.generate(n, w, t, 1.0, seed=7, tile_size=b)
    assert tib.two_chain_order(m)[1] > 0
    res = tib.selected_inverse(m, "pattern")
    assert np.max(np.abs(res.diagonal() - ref["diag"]) / np.abs(ref["diag"])) <= 1e-10
    assert abs(res.logdet() - ref["logdet"]) <= 1e-10 * abs(ref["logdet"])
    ms = [m] + [tib.generate(n, w, t, 1.0, seed=100 + k, tile_size=b) for k in range(32)]
    logdet, diag = tib.selected_inverse_batch(ms)
    assert np.max(np.abs(diag[0] - ref["diag"]) / np.abs(ref["diag"])) <= 1e-10
    assert abs(logdet[0] - ref["logdet"]) <= 1e-10 * abs(ref["logdet"])
