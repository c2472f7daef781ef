"""Host-side logic of the product library, CPU only (no compute calls): the
C ABI loads and exports every declared symbol, the symbolic planner is
tile-for-tile identical to the reference's, the input side (generator,
from_dense, Matrix Market) is bit-exact, errors map like the reference, and
the task-model FLOP counts match the reference driver's."""
import ctypes
import json
import os
import re
import subprocess

import numpy as np
import pytest

from conftest import GOLDEN, REF_DRIVER, ROOT


def declared_symbols():
    text = open(os.path.join(ROOT, "include", "tileinv_b200.h")).read()
    return sorted(set(re.findall(r"\b(tib_[a-z0-9_]+)\s*\(", text)))


def test_c_abi_exports_every_declared_symbol(tib):
    from paper_2504_19171_b200 import _lib

    lib = ctypes.CDLL(_lib.LIB_PATH)
    names = declared_symbols()
    assert len(names) >= 35
    for name in names:
        assert hasattr(lib, name), name
    # the Python binding covers every C entry point
    assert set(names) == set(_lib.EXPORTED)


def test_library_is_sm100a_only():
    from paper_2504_19171_b200 import _lib

    out = subprocess.run(["cuobjdump", "-lelf", _lib.LIB_PATH], capture_output=True, text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    assert "sm_100a" in out.stdout
    sass = subprocess.run(["cuobjdump", "-sass", _lib.LIB_PATH], capture_output=True, text=True).stdout
    assert "DMMA.8x8x4" in sass  # FP64 tensor-core path


def test_symbolic_matches_reference(tib):
    cases = json.load(open(os.path.join(GOLDEN, "symbolic.json")))
    for key, case in cases.items():
        n, w, t, d, seed, b, sel = case["args"]
        if not isinstance(sel, str):
            sel = [tuple(p) for p in sel]
        m = tib.generate(n, w, t, d, seed=seed, tile_size=b)
        assert tib.factor_pattern(m) == [tuple(x) for x in case["factor"]], key
        closure, growth = tib.closure_tiles(m, sel)
        assert closure == [tuple(x) for x in case["closure"]], key
        assert growth == case["growth_warning"], key


@pytest.mark.skipif(not os.path.exists(REF_DRIVER), reason="oracle/_ref not built")
@pytest.mark.parametrize("args", [
    (10000, 200, 50, 128, 42, 1.0, "pattern"),
    (5000, 700, 9, 256, 1, 0.05, "diagonal"),
    (3000, 300, 40, 100, 8, 1.0, "all"),
    (2000, 100, 0, 64, 3, 1.0, "1999,0;1000,999;0,0"),
])
def test_symbolic_matches_live_reference(tib, args):
    n, w, t, b, seed, d, sel = args
    out = json.loads(subprocess.run([REF_DRIVER, "symbolic", str(n), str(w), str(t), str(b), str(seed), repr(d), sel],
                                    check=True, capture_output=True, text=True).stdout)
    m = tib.generate(n, w, t, d, seed=seed, tile_size=b)
    if sel not in ("pattern", "diagonal", "all"):
        sel = [tuple(int(v) for v in p.split(",")) for p in sel.split(";")]
    assert tib.factor_pattern(m) == [tuple(x) for x in out["factor"]]
    assert tib.closure_tiles(m, sel)[0] == [tuple(x) for x in out["closure"]]


def test_generator_bit_exact(tib, ref):
    for (n, w, t, d, seed, b) in [(24, 5, 2, 0.8, 7, 4), (1000, 150, 20, 1.0, 13, 128), (777, 64, 0, 0.3, 4, 50)]:
        ours = tib.generate(n, w, t, d, seed=seed, tile_size=b)
        theirs = ref.generate(n, w, t, d, seed=seed, tile_size=b)
        assert ours.stored_tiles == theirs.stored_tiles
        assert np.array_equal(ours.to_dense(), theirs.to_dense())


def test_matrix_market_round_trip_is_byte_identical(tib, ref, tmp_path):
    m_ours = tib.generate(200, 30, 5, 0.6, seed=3, tile_size=16)
    m_ref = ref.generate(200, 30, 5, 0.6, seed=3, tile_size=16)
    tib.write_matrix_market(m_ours, str(tmp_path / "ours.mtx"))
    ref.write_matrix_market(m_ref, str(tmp_path / "ref.mtx"))
    assert (tmp_path / "ours.mtx").read_bytes() == (tmp_path / "ref.mtx").read_bytes()
    back = tib.read_matrix_market(str(tmp_path / "ref.mtx"), tile_size=24)
    assert np.array_equal(back.to_dense(), m_ref.to_dense())


def test_from_dense_and_padding(tib, ref):
    rng = np.random.default_rng(0)
    a = rng.standard_normal((37, 37))
    a = a @ a.T + 37 * np.eye(37)
    a[np.abs(a) < 0.5] = 0.0
    ours, theirs = tib.from_dense(a, tile_size=8), ref.from_dense(a, tile_size=8)
    assert ours.n_tiles == theirs.n_tiles == 5 and ours.stored_tiles == theirs.stored_tiles
    assert np.array_equal(ours.to_dense(), theirs.to_dense())
    ti, tj, pay = ours.tiles()
    last = pay[list(zip(ti, tj)).index((4, 4))]
    assert np.array_equal(np.diag(last)[5:], np.ones(3))  # identity on the padded rows


def test_errors_map_like_the_reference(tib, tmp_path):
    with pytest.raises(tib.TileinvError, match="n must be positive"):  # matgen.cpp:46
        tib.generate(0, 1, 0, 1.0)
    with pytest.raises(tib.TileinvError, match="thickness"):
        tib.generate(10, 2, 10, 1.0)
    with pytest.raises(tib.TileinvError, match="density"):
        tib.generate(10, 2, 1, 0.0)
    with pytest.raises(ValueError):
        tib.from_dense(np.zeros((2, 3)))
    with pytest.raises(ValueError):
        tib.closure_tiles(tib.generate(10, 2, 1, 1.0, tile_size=2), "bogus")
    with pytest.raises(tib.TileinvError, match="outside the matrix"):
        tib.closure_tiles(tib.generate(10, 2, 1, 1.0, tile_size=2), [(10, 0)])
    bad = tmp_path / "bad.mtx"
    bad.write_text("%%MatrixMarket matrix coordinate real general\n2 2 1\n1 1 1.0\n")
    with pytest.raises(tib.TileinvError, match="only symmetric"):
        tib.read_matrix_market(str(bad))
    bad.write_text("%%MatrixMarket matrix coordinate real symmetric\n2 2 1\n1 2 1.0\n")
    with pytest.raises(tib.TileinvError, match="upper-triangle"):
        tib.read_matrix_market(str(bad))
    with pytest.raises(tib.TileinvError, match="cannot open"):
        tib.read_matrix_market(str(tmp_path / "missing.mtx"))
    with pytest.raises(tib.TileinvError, match="worker count"):
        tib.factorize(tib.generate(10, 2, 1, 1.0, tile_size=2), workers=0)


def test_task_model_flops_match_reference_driver(tib):
    g = np.load(os.path.join(GOLDEN, "small.npz"))
    f, p1, p2 = tib.task_flops(tib.generate(10000, 200, 50, 1.0, seed=42, tile_size=128))
    assert abs(f / 1e9 - float(g["gflop_factorize"])) < 1e-6
    assert abs(p1 / 1e9 - float(g["gflop_phase1"])) < 1e-6
    assert abs(p2 / 1e9 - float(g["gflop_phase2"])) < 1e-6
    # SURVEY.md Appendix B, large (b=512): 1577.1 / 277.9 / 3136.7 GFLOP
    f, p1, p2 = tib.task_flops(tib.generate(200000, 2000, 200, 1.0, seed=42, tile_size=512))
    assert round(f / 1e9, 1) == 1577.1 and round(p1 / 1e9, 1) == 277.9 and round(p2 / 1e9, 1) == 3136.7


def test_no_cuda_device_fails_loudly(tib):
    if tib.device_count() > 0:
        pytest.skip("a GPU is present")
    with pytest.raises(tib.TileinvError, match="no CPU fallback"):
        tib.selected_inverse(tib.generate(10, 2, 1, 1.0, tile_size=2))


def test_two_chain_order(tib):
    """Two-chain elimination order (planner.cpp two_chain_order): a permutation
    [I_0 ascending, I_1 descending, separator, arrow] whose symbolic fill adds
    no tile, or none at all when the pattern does not admit one."""
    for n, w, t, b in ((3000, 200, 30, 64), (200000, 2000, 200, 512), (100000, 1000, 100, 256), (4096, 300, 0, 128)):
        m = tib.generate(n, w, t, 1.0, seed=1, tile_size=b)
        order, split = tib.two_chain_order(m)
        N = m.n_tiles
        assert split > 0 and sorted(order.tolist()) == list(range(N))
        # the arrow stays last (no arrow: the separator is last); I_0 is the identity prefix
        assert order[-1] == N - 1 if t else order[-1] < N - 1
        assert order[:split].tolist() == list(range(split))
        # the second chain starts at the far end of the band and descends
        assert order[split] > order[split + 1]
        mp = tib.two_chain_permuted(m)
        assert mp.stored_tiles == len(tib.factor_pattern(m)) == len(tib.factor_pattern(mp))
    # too few tile columns for two interiors and a separator, and a partial last
    # band tile with no arrow (it would fill in across the second interior)
    assert tib.two_chain_order(tib.generate(700, 300, 0, 1.0, seed=1, tile_size=64))[1] == -1
    assert tib.two_chain_order(tib.generate(4000, 300, 0, 1.0, seed=1, tile_size=128))[1] == -1
