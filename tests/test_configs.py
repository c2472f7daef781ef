"""Parity at the BASELINE configs themselves (SURVEY.md 8(c) gate, per config),
against numbers the REFERENCE produced on the same inputs (tests/golden/
config_*.npz, written by `make_golden.py configs` from `ref_driver golden`:
the unmodified reference's factorize + phase1 + phase2).

  config 2 medium  n=100000 w=1000 t=100 b=256 seed 42
  config 3 large   n=200000 w=2000 t=200 b=512 seed 42
  config 5 batch   64 x (n=50000 w=500 t=50) b=128 seeds 1000..1063 (members
                   1000 and 1063 pinned)
  config 4 Kronecker AR1 x SPDE + 20 fixed effects at reduced scale (10 x
                   20x20 sites, b=128; 50 x 40x25 sites, b=256), given to the
                   reference as Matrix Market (read_matrix_market_file)

Checked: diag(Sigma) elementwise <= 1e-10, logdet relative <= 1e-10, the
closure tile count, per closure tile the Frobenius norm (relative <= 1e-10),
the plain and weighted sums (within 1e-10 of the tile's b * Frobenius norm),
and sampled 64 x 64 blocks of the last three tile columns, the middle column
and the arrow normwise <= 1e-10.  The input matrices are pinned bit-for-bit
by the reference's payload_checksum (host generator on CPU; the device
generator on the GPU)."""
import os

import numpy as np
import pytest

from conftest import GOLDEN, elementwise

TOL = 1e-10


def golden(name):
    return np.load(os.path.join(GOLDEN, f"config_{name}.npz"))


@pytest.mark.parametrize("name", ["medium", "batch1000", "batch1063"])
def test_host_generator_checksum_equals_reference(tib, name):
    g = golden(name)
    n, w, t, b, seed = (int(x) for x in g["args"])
    assert tib.generate(n, w, t, 1.0, seed=seed, tile_size=b).checksum == int(g["matrix_checksum"])


@pytest.mark.parametrize("name", ["kron_small", "kron_mid"])
def test_kronecker_generator_checksum_equals_reference(tib, name):
    """The reference read our Matrix Market file of this matrix and computed
    the same payload_checksum: generator + writer pinned byte for byte."""
    g = golden(name)
    nt, nx, ny, p, b = (int(x) for x in g["args"])
    assert tib.generate_kronecker(nt, nx, ny, p, tile_size=b).checksum == int(g["matrix_checksum"])


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["kron_small", "kron_mid"])
def test_kronecker_config_vs_reference(tib, name):
    g = golden(name)
    nt, nx, ny, p, b = (int(x) for x in g["args"])
    m = tib.generate_kronecker(nt, nx, ny, p, tile_size=b)
    res = tib.selected_inverse(m, "pattern")
    ti, tj, pay = res.tiles()
    check_against_golden(g, m.n, b, res.diagonal(), res.logdet(), ti, tj, pay)


def tile_stats(pay):
    b = pay.shape[1]
    r = np.arange(b)[:, None]
    c = np.arange(b)[None, :]
    wgt = ((7 * r + 13 * c) % 11 - 5).astype(np.float64)
    fro = np.sqrt(np.einsum("kij,kij->k", pay, pay))
    return np.stack([fro, pay.sum(axis=(1, 2)), np.einsum("kij,ij->k", pay, wgt)], 1)


def check_against_golden(g, n, b, diag, logdet, ti, tj, pay):
    assert elementwise(diag, g["diag"]) <= TOL
    assert abs(logdet - float(g["logdet"])) <= TOL * abs(float(g["logdet"]))
    if pay is None:
        return
    assert len(ti) == int(g["closure_tiles"])
    st, ref = tile_stats(pay), g["tstats"]
    assert np.all(np.abs(st[:, 0] - ref[:, 0]) <= TOL * ref[:, 0])
    bound = TOL * b * ref[:, 0]
    assert np.all(np.abs(st[:, 1] - ref[:, 1]) <= bound)
    assert np.all(np.abs(st[:, 2] - ref[:, 2]) <= 5 * bound)
    slot = {(int(i), int(j)): k for k, (i, j) in enumerate(zip(ti, tj))}
    s = g["blocks"].shape[-1]
    scale = np.abs(g["blocks"]).max()
    for (i, j), ref_blk in zip(g["sampled"], g["blocks"]):
        tile = pay[slot[(int(i), int(j))]]
        vr, vc = min(b, n - int(i) * b), min(b, n - int(j) * b)
        r0, c0 = max(0, vr - s), max(0, vc - s)
        got = (tile[:s, :s], tile[r0:r0 + s, c0:c0 + s])
        for part in range(2):
            assert np.abs(got[part] - ref_blk[part]).max() <= TOL * scale, (i, j, part)


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["medium", "large"])
def test_single_matrix_config_vs_reference(tib, name):
    g = golden(name)
    n, w, t, b, seed = (int(x) for x in g["args"])
    m = tib.generate(n, w, t, 1.0, seed=seed, tile_size=b, device=0)
    res = tib.selected_inverse(m, "pattern")
    ti, tj, pay = res.tiles()
    check_against_golden(g, n, b, res.diagonal(), res.logdet(), ti, tj, pay)
    del pay
    # the device generator made exactly the reference's matrix
    assert m.checksum == int(g["matrix_checksum"])


@pytest.mark.gpu
def test_batch_config_vs_reference(tib, monkeypatch):
    """BASELINE config 5 as one batched call: 64 device-generated matrices;
    the first and last members against the reference's own runs."""
    ms = [tib.generate(50000, 500, 50, 1.0, seed=1000 + k, tile_size=128, device=0) for k in range(64)]
    logdet, diag = tib.selected_inverse_batch(ms)
    for k, name in ((0, "batch1000"), (63, "batch1063")):
        check_against_golden(golden(name), 50000, 128, diag[k], logdet[k], None, None, None)
    # members are independent: one member alone (in the natural elimination
    # order, like the batch) gives the same bits
    # (a batch runs plain leaf tasks, groups its bulk updates four to a task and
    # phase 2's late terms eight to a part; a single call runs the chain task:
    # the same values to rounding)
    monkeypatch.setenv("TIB_SPLIT", "0")
    single = tib.selected_inverse(ms[63], "pattern")
    assert abs(single.logdet() - logdet[63]) <= 1e-14 * abs(logdet[63])
    assert elementwise(single.diagonal(), diag[63]) <= 1e-13


@pytest.mark.gpu
def test_device_generator_is_bitwise_the_host_generator(tib, monkeypatch):
    # (one elimination order for both: host matrices may stream in the natural one)
    monkeypatch.setenv("TIB_SPLIT", "0")
    for args in ((10000, 200, 50, 42, 128), (5000, 0, 700, 3, 96), (3000, 400, 0, 9, 100), (777, 50, 30, 1, 64)):
        n, w, t, seed, b = args
        h = tib.generate(n, w, t, 1.0, seed=seed, tile_size=b)
        d = tib.generate(n, w, t, 1.0, seed=seed, tile_size=b, device=0)
        for x, y in zip(h.tiles(), d.tiles()):
            assert np.array_equal(x, y), args
        assert h.checksum == d.checksum
        rh = tib.selected_inverse(h, "pattern")
        rd = tib.selected_inverse(d, "pattern")
        assert rh.checksum == rd.checksum
