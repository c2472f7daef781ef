"""STLS tile files (the reference's checkpoint / resume format,
/root/reference/proj/src/tileio.cpp:30-94) against files the REFERENCE wrote
itself (tests/golden/stls/, `ref_driver stls`: write_tile_file of the
generated matrix, of factorize's L, of phase1's U / W, and
write_selected_inverse of the pattern inverse).

CPU: the matrix file we write is byte-identical to the reference's; we read
the reference's files; malformed files fail like the reference (ParseError ->
TileinvError; a file of the wrong phase -> TileinvError).
GPU: a factor read from the reference's kFactor or kPhase1 file (the CLI's
`selinv --factor`, tileinv_main.cpp:183-185) gives the reference's Sigma;
our factor / phase-1 / Sigma files carry the reference's header and tile
list, payload within the parity gate."""
import gzip
import os
import struct

import numpy as np
import pytest

from conftest import GOLDEN, normwise

STLS = os.path.join(GOLDEN, "stls")
CASES = {"case_b32": (200, 30, 6, 32, 4), "case_b100": (250, 30, 6, 100, 3)}  # make_golden.STLS_CASES
TOL = 1e-10


def ref_bytes(name, kind):
    with gzip.open(os.path.join(STLS, f"{name}.{kind}.stls.gz"), "rb") as f:
        return f.read()


def ref_file(tmp_path, name, kind):
    p = tmp_path / f"{name}.{kind}.stls"
    p.write_bytes(ref_bytes(name, kind))
    return str(p)


def parse(data):
    assert data[:4] == b"STLS"
    version, n, b, N, phase, count = struct.unpack_from("<6I", data, 4)
    off, tiles, pay = 28, [], []
    for _ in range(count):
        i, j = struct.unpack_from("<2I", data, off)
        off += 8
        pay.append(np.frombuffer(data, np.float64, b * b, off).reshape(b, b))
        off += 8 * b * b
        tiles.append((i, j))
    assert off == len(data)
    return {"version": version, "n": n, "b": b, "N": N, "phase": phase, "tiles": tiles, "payload": np.array(pay)}


@pytest.mark.parametrize("name", sorted(CASES))
def test_matrix_file_is_byte_identical(tib, tmp_path, name):
    n, w, t, b, seed = CASES[name]
    out = tmp_path / "m.stls"
    tib.generate(n, w, t, 1.0, seed=seed, tile_size=b).write_tiles(str(out))
    assert out.read_bytes() == ref_bytes(name, "matrix")


@pytest.mark.parametrize("name", sorted(CASES))
def test_read_reference_matrix_file(tib, tmp_path, name):
    n, w, t, b, seed = CASES[name]
    m = tib.read_matrix_tiles(ref_file(tmp_path, name, "matrix"))
    g = tib.generate(n, w, t, 1.0, seed=seed, tile_size=b)
    assert (m.n, m.tile_size, m.stored_tiles) == (n, b, g.stored_tiles)
    assert m.checksum == g.checksum


def test_malformed_files(tib, tmp_path):
    good = ref_bytes("case_b32", "matrix")
    cases = {
        "magic": b"STLX" + good[4:],
        "version": good[:4] + struct.pack("<I", 2) + good[8:],
        "truncated": good[:-100],
        "grid": good[:16] + struct.pack("<I", 99) + good[20:],
        "phase": good[:20] + struct.pack("<I", 7) + good[24:],
        "upper": good[:28] + struct.pack("<2I", 0, 1) + good[36:],
    }
    for what, data in cases.items():
        p = tmp_path / f"{what}.stls"
        p.write_bytes(data)
        with pytest.raises(tib.TileinvError):
            tib.read_matrix_tiles(str(p))
    with pytest.raises(tib.TileinvError, match="cannot open"):
        tib.read_matrix_tiles(str(tmp_path / "missing.stls"))
    # a factor file is not a matrix file (FormatError, tileio.cpp:99-105)
    with pytest.raises(tib.TileinvError, match="expected a matrix tile file"):
        tib.read_matrix_tiles(ref_file(tmp_path, "case_b32", "factor"))


@pytest.mark.gpu
@pytest.mark.parametrize("name", sorted(CASES))
@pytest.mark.parametrize("kind", ["factor", "phase1"])
def test_selected_inverse_from_reference_factor_file(tib, tmp_path, name, kind):
    f = tib.read_factor_tiles(ref_file(tmp_path, name, kind))
    assert f.phase == (1 if kind == "factor" else 2)
    res = tib.selected_inverse_of_factor(f, "pattern")
    sig = parse(ref_bytes(name, "sigma"))
    ti, tj, pay = res.tiles()
    assert list(zip(ti.tolist(), tj.tolist())) == sig["tiles"]
    assert normwise(pay, sig["payload"]) <= TOL
    n, w, t, b, seed = CASES[name]
    direct = tib.selected_inverse(tib.generate(n, w, t, 1.0, seed=seed, tile_size=b), "pattern")
    assert abs(f.logdet() - direct.logdet()) <= TOL * abs(direct.logdet())
    if kind == "phase1":
        with pytest.raises(tib.TileinvError):
            f.tiles(1)


@pytest.mark.gpu
@pytest.mark.parametrize("name", sorted(CASES))
def test_written_files_match_reference_files(tib, tmp_path, name):
    n, w, t, b, seed = CASES[name]
    m = tib.generate(n, w, t, 1.0, seed=seed, tile_size=b)
    f = tib.factorize(m)
    f.write_tiles(str(tmp_path / "f.stls"), phase=1)
    f.write_tiles(str(tmp_path / "p1.stls"), phase=2)
    tib.selected_inverse(m, "pattern").write_tiles(str(tmp_path / "s.stls"))
    for ours, kind in (("f.stls", "factor"), ("p1.stls", "phase1"), ("s.stls", "sigma")):
        a, r = parse((tmp_path / ours).read_bytes()), parse(ref_bytes(name, kind))
        assert {k: a[k] for k in ("version", "n", "b", "N", "phase", "tiles")} == \
               {k: r[k] for k in ("version", "n", "b", "N", "phase", "tiles")}, kind
        assert normwise(a["payload"], r["payload"]) <= TOL, kind
    # round trip: our own files resume to the same result
    again = tib.selected_inverse_of_factor(tib.read_factor_tiles(str(tmp_path / "f.stls")), "pattern")
    assert normwise(again.tiles()[2], parse(ref_bytes(name, "sigma"))["payload"]) <= TOL
