"""B200-native drop-in for the hot path of ``tileinv`` (arXiv 2504.19171, sTiles).

Same names, argument meaning and error behaviour as the reference Python
module (proj/bindings/module.cpp:125-237, proj/python/tileinv/__init__.py):

    Matrix, Factor, SelectedInverseResult, TileinvError, NotSpdError,
    generate, from_dense, read_matrix_market, write_matrix_market,
    factorize, selected_inverse, selected_inverse_of_factor

Everything numeric runs through the C ABI of ``libtileinv_b200.so``
(include/tileinv_b200.h): the tile Cholesky, the phase-1 transform and the
phase-2 Takahashi recursion are sm_100a kernels on the GPU, the factor and
the result stay resident in HBM.  ``workers`` is accepted for compatibility
(it must be >= 1, like the reference); ``device`` picks the GPU.

Additions beyond the reference API: ``Factor.logdet()``, ``Factor.tiles()``,
``SelectedInverseResult.diagonal()`` (marginal variances as a numpy array),
``.logdet()``, ``.tiles()``, ``selected_inverse_batch`` and the symbolic
helpers ``factor_pattern`` / ``closure_tiles`` / ``task_flops``.

The DAG analyzer (dag_report / export_dot / predict_gemm_count) is outside
this path (component 10) and is not provided.
"""
from __future__ import annotations

import ctypes as C
from typing import Iterable, Sequence

import numpy as np

from ._lib import lib

__version__ = lib.tib_version().decode()

_PRESETS = {"diagonal": 1, "pattern": 2, "all": 3}
_ORACLE_LIMIT = 4000  # proj/include/tileinv/oracle.hpp:22


class TileinvError(RuntimeError):
    """Any reference ``tileinv::Error`` (module.cpp:131)."""


class NotSpdError(ArithmeticError):
    """``tileinv::NotSpdError`` (module.cpp:132); carries pivot / tile."""

    def __init__(self, msg: str, pivot: int = -1, tile_i: int = -1, tile_j: int = -1):
        super().__init__(msg)
        self.pivot = pivot
        self.tile_i = tile_i
        self.tile_j = tile_j


def _check(status: int) -> None:
    if status == 0:
        return
    msg = lib.tib_last_error_message().decode(errors="replace")
    if status == 3:
        pivot, ti, tj = C.c_long(), C.c_int(), C.c_int()
        lib.tib_last_not_spd(C.byref(pivot), C.byref(ti), C.byref(tj))
        raise NotSpdError(msg, pivot.value, ti.value, tj.value)
    raise TileinvError(msg)


def _request(selection) -> tuple[int, np.ndarray | None, np.ndarray | None, int]:
    """module.cpp:34-44: a preset name or a list of (r, c) pairs."""
    if isinstance(selection, str):
        if selection not in _PRESETS:
            raise ValueError("selection must be 'diagonal', 'pattern', 'all', or a pair list")
        return _PRESETS[selection], None, None, 0
    pairs = [(int(r), int(c)) for r, c in selection]
    rows = np.ascontiguousarray([p[0] for p in pairs], dtype=np.int64)
    cols = np.ascontiguousarray([p[1] for p in pairs], dtype=np.int64)
    return 0, rows, cols, len(pairs)


def _lp(a):
    return None if a is None else a.ctypes.data_as(C.POINTER(C.c_long))


def _check_workers(workers: int) -> None:
    if workers < 1:
        raise TileinvError("worker count must be at least 1")


class Matrix:
    """TiledSymmetricMatrix (storage.hpp:40-44), host resident."""

    def __init__(self, handle: int):
        self._h = C.c_void_p(handle)

    def __del__(self, _free=lib.tib_matrix_free):  # bound now: module globals are gone at interpreter exit
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            _free(h)
            self._h = None

    def _info(self):
        n, b, N, s = C.c_long(), C.c_int(), C.c_int(), C.c_long()
        _check(lib.tib_matrix_info(self._h, C.byref(n), C.byref(b), C.byref(N), C.byref(s)))
        return n.value, b.value, N.value, s.value

    @property
    def n(self) -> int:
        return self._info()[0]

    @property
    def tile_size(self) -> int:
        return self._info()[1]

    @property
    def n_tiles(self) -> int:
        return self._info()[2]

    @property
    def stored_tiles(self) -> int:
        return self._info()[3]

    def tiles(self):
        """(ti, tj, payload[count, b, b]) in column-major tile order."""
        n, b, N, s = self._info()
        ti = np.empty(s, np.int32)
        tj = np.empty(s, np.int32)
        pay = np.empty((s, b, b), np.float64)
        _check(lib.tib_matrix_tiles(self._h, ti.ctypes.data_as(C.POINTER(C.c_int)),
                                    tj.ctypes.data_as(C.POINTER(C.c_int)),
                                    pay.ctypes.data_as(C.POINTER(C.c_double))))
        return ti, tj, pay

    @property
    def checksum(self) -> int:
        """payload_checksum (storage.cpp:34-48) of the tiles: equals the
        reference's value for the same matrix."""
        out = C.c_uint64()
        _check(lib.tib_matrix_checksum(self._h, C.byref(out)))
        return out.value

    def write_tiles(self, path: str) -> None:
        """STLS tile file, kMatrix (write_tile_file, tileio.cpp:30-53)."""
        _check(lib.tib_matrix_write_stls(self._h, path.encode()))

    def to_dense(self) -> np.ndarray:
        """dense_from_tiled (oracle.cpp:24-45), with the reference's n <= 4000 guard."""
        n, b, N, s = self._info()
        if n > _ORACLE_LIMIT:
            raise TileinvError(f"oracle limited to n <= {_ORACLE_LIMIT}, got n = {n}")
        ti, tj, pay = self.tiles()
        return _tiles_to_dense(n, b, ti, tj, pay)


class Factor:
    """TiledFactor (storage.hpp:46-51); device resident (L and the phase-1 tiles)."""

    def __init__(self, handle: int):
        self._h = C.c_void_p(handle)

    def __del__(self, _free=lib.tib_factor_free):  # bound now: module globals are gone at interpreter exit
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            _free(h)
            self._h = None

    def _info(self):
        n, b, s = C.c_long(), C.c_int(), C.c_long()
        _check(lib.tib_factor_info(self._h, C.byref(n), C.byref(b), C.byref(s)))
        return n.value, b.value, s.value

    @property
    def n(self) -> int:
        return self._info()[0]

    @property
    def tile_size(self) -> int:
        return self._info()[1]

    @property
    def stored_tiles(self) -> int:
        return self._info()[2]

    @property
    def checksum(self) -> int:
        out = C.c_uint64()
        _check(lib.tib_factor_checksum(self._h, C.byref(out)))
        return out.value

    def logdet(self) -> float:
        out = C.c_double()
        _check(lib.tib_factor_logdet(self._h, C.byref(out)))
        return out.value

    @property
    def phase(self) -> int:
        """PhaseTag of the held tiles: 1 kFactor (L + phase-1 tiles), 2 kPhase1."""
        out = C.c_int()
        _check(lib.tib_factor_phase(self._h, C.byref(out)))
        return out.value

    def write_tiles(self, path: str, phase: int = 1) -> None:
        """STLS tile file (write_tile_file, tileio.cpp:30-53): phase 1 writes L
        (kFactor), phase 2 the phase-1 tiles U / W (kPhase1)."""
        _check(lib.tib_factor_write_stls(self._h, phase, path.encode()))

    def tiles(self, phase: int = 1):
        """phase 1: L tiles; phase 2: phase-1 tiles (U on the diagonal, W off it)."""
        n, b, s = self._info()
        ti = np.empty(s, np.int32)
        tj = np.empty(s, np.int32)
        pay = np.empty((s, b, b), np.float64)
        _check(lib.tib_factor_tiles(self._h, phase, ti.ctypes.data_as(C.POINTER(C.c_int)),
                                    tj.ctypes.data_as(C.POINTER(C.c_int)),
                                    pay.ctypes.data_as(C.POINTER(C.c_double))))
        return ti, tj, pay

    def get_tiles(self, coords) -> np.ndarray:
        """The L tiles at `coords` [(i, j), ...] as a (k, b, b) array."""
        ti, tj = _coords(coords)
        b = self.tile_size
        pay = np.empty((len(ti), b, b), np.float64)
        _check(lib.tib_factor_get_tiles(self._h, len(ti), ti.ctypes.data_as(C.POINTER(C.c_int)),
                                        tj.ctypes.data_as(C.POINTER(C.c_int)),
                                        pay.ctypes.data_as(C.POINTER(C.c_double))))
        return pay

    def replace_tiles(self, coords, payload) -> None:
        """Overwrites L tiles on the device and recomputes the phase-1 tiles and
        logdet (the partitioned path: the border block of a rank's system)."""
        ti, tj = _coords(coords)
        pay = np.ascontiguousarray(payload, np.float64)
        b = self.tile_size
        if pay.shape != (len(ti), b, b):
            raise ValueError(f"payload shape {pay.shape} != {(len(ti), b, b)}")
        _check(lib.tib_factor_replace_tiles(self._h, len(ti), ti.ctypes.data_as(C.POINTER(C.c_int)),
                                            tj.ctypes.data_as(C.POINTER(C.c_int)),
                                            pay.ctypes.data_as(C.POINTER(C.c_double))))


def _coords(coords):
    c = np.asarray(coords, np.int32).reshape(-1, 2)
    return np.ascontiguousarray(c[:, 0]), np.ascontiguousarray(c[:, 1])


class SelectedInverseResult:
    """SelectedInverse (selinv.hpp:61-68) + its request; device resident."""

    def __init__(self, handle: int):
        self._h = C.c_void_p(handle)

    def __del__(self, _free=lib.tib_sigma_free):  # bound now: module globals are gone at interpreter exit
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            _free(h)
            self._h = None

    def _info(self):
        n, b, t, g = C.c_long(), C.c_int(), C.c_long(), C.c_int()
        _check(lib.tib_sigma_info(self._h, C.byref(n), C.byref(b), C.byref(t), C.byref(g)))
        return n.value, b.value, t.value, g.value

    @property
    def n(self) -> int:
        return self._info()[0]

    @property
    def closure_tiles(self) -> int:
        return self._info()[2]

    @property
    def growth_warning(self) -> bool:
        return bool(self._info()[3])

    @property
    def checksum(self) -> int:
        out = C.c_uint64()
        _check(lib.tib_sigma_checksum(self._h, C.byref(out)))
        return out.value

    def write_tiles(self, path: str) -> None:
        """write_selected_inverse (selinv.cpp:441): the closure tiles as an STLS
        file tagged kSelectedInverse."""
        _check(lib.tib_sigma_write_stls(self._h, path.encode()))

    def entries_arrays(self):
        """extract_entries (selinv.cpp:387-439) as (rows, cols, values) numpy arrays."""
        cnt = C.c_long()
        _check(lib.tib_sigma_entries(self._h, C.byref(cnt), None, None, None))
        rows = np.empty(cnt.value, np.int64)
        cols = np.empty(cnt.value, np.int64)
        vals = np.empty(cnt.value, np.float64)
        _check(lib.tib_sigma_entries(self._h, C.byref(cnt), _lp(rows), _lp(cols),
                                     vals.ctypes.data_as(C.POINTER(C.c_double))))
        return rows, cols, vals

    def entries(self):
        """List of (r, c, value) tuples, like module.cpp:154-161."""
        rows, cols, vals = self.entries_arrays()
        return [(int(r), int(c), float(v)) for r, c, v in zip(rows.tolist(), cols.tolist(), vals.tolist())]

    def diagonal(self) -> np.ndarray:
        """Marginal variances diag(Sigma), written by the phase-2 diagonal kernel."""
        n = self._info()[0]
        out = np.empty(n, np.float64)
        _check(lib.tib_sigma_diagonal(self._h, out.ctypes.data_as(C.POINTER(C.c_double))))
        return out

    def logdet(self) -> float:
        out = C.c_double()
        _check(lib.tib_sigma_logdet(self._h, C.byref(out)))
        return out.value

    def tiles(self):
        n, b, t, _ = self._info()
        ti = np.empty(t, np.int32)
        tj = np.empty(t, np.int32)
        pay = np.empty((t, b, b), np.float64)
        _check(lib.tib_sigma_tiles(self._h, ti.ctypes.data_as(C.POINTER(C.c_int)),
                                   tj.ctypes.data_as(C.POINTER(C.c_int)),
                                   pay.ctypes.data_as(C.POINTER(C.c_double))))
        return ti, tj, pay

    def to_dense(self) -> np.ndarray:
        """result_to_dense (module.cpp:83-107): zeros outside the closure."""
        n, b, t, _ = self._info()
        ti, tj, pay = self.tiles()
        return _tiles_to_dense(n, b, ti, tj, pay)


def _tiles_to_dense(n, b, ti, tj, pay) -> np.ndarray:
    """Symmetric dense expansion of lower tiles (r >= c kept, mirrored)."""
    out = np.zeros((n, n))
    for k in range(len(ti)):
        r0, c0 = int(ti[k]) * b, int(tj[k]) * b
        nr, nc = max(0, min(b, n - r0)), max(0, min(b, n - c0))
        if nr == 0 or nc == 0:
            continue
        rows = np.broadcast_to(np.arange(nr)[:, None] + r0, (nr, nc))
        cols = np.broadcast_to(np.arange(nc)[None, :] + c0, (nr, nc))
        keep = cols <= rows
        out[rows[keep], cols[keep]] = pay[k][:nr, :nc][keep]
    il = np.tril_indices(n, -1)
    out[il[1], il[0]] = out[il]
    return out


def _new_handle() -> C.c_void_p:
    return C.c_void_p()


def generate(n: int, bandwidth: int, thickness: int, density: float, seed: int = 0,
             tile_size: int = 32, device: int | None = None) -> Matrix:
    """generate_arrowhead (matgen.cpp:59-120), bit-exact values.

    ``device=k`` (density 1 only): the values are generated on GPU k straight
    into each sweep's tile store (generate.cu) -- no host payload, no H2D copy;
    ``tiles()`` / ``checksum`` / ``write_matrix_market`` read them back from
    the device."""
    h = _new_handle()
    if device is None:
        _check(lib.tib_matrix_generate(n, bandwidth, thickness, float(density), seed, tile_size, C.byref(h)))
    else:
        if float(density) != 1.0:
            raise TileinvError("device generation needs density 1 (the draw index is closed-form only there)")
        _check(lib.tib_matrix_generate_device(n, bandwidth, thickness, seed, tile_size, device, C.byref(h)))
    return Matrix(h.value)


# BASELINE config 4: 50 time steps x 4000 sites (80 x 50 lattice) + 20 fixed effects
KRONECKER_CONFIG = dict(nt=50, nx=80, ny=50, p=20, rho=0.9, kappa2=0.5, tau=1.0, tau_y=1.0, q_beta=0.01, seed=42)


def generate_kronecker(nt: int, nx: int, ny: int, p: int, rho: float = 0.9, kappa2: float = 0.5, tau: float = 1.0,
                       tau_y: float = 1.0, q_beta: float = 0.01, seed: int = 42, tile_size: int = 32) -> Matrix:
    """Spatio-temporal Kronecker arrowhead (BASELINE config 4; kronecker.cpp):
    joint precision of an AR1(rho) x SPDE(nx x ny lattice) latent field (time
    major) and p fixed effects, the dense arrow.  The reference cannot generate
    it; it reads it through Matrix Market (``write_matrix_market``)."""
    h = _new_handle()
    _check(lib.tib_matrix_generate_kronecker(nt, nx, ny, p, float(rho), float(kappa2), float(tau), float(tau_y),
                                             float(q_beta), seed, tile_size, C.byref(h)))
    return Matrix(h.value)


def from_dense(array, tile_size: int = 32) -> Matrix:
    a = np.ascontiguousarray(array, dtype=np.float64)
    if a.ndim != 2 or a.shape[0] != a.shape[1]:
        raise ValueError("from_dense needs a square 2-D array")
    h = _new_handle()
    _check(lib.tib_matrix_from_dense(a.shape[0], tile_size, a.ctypes.data_as(C.POINTER(C.c_double)),
                                     C.byref(h)))
    return Matrix(h.value)


def from_tiles(n: int, tile_size: int, ti: Sequence[int], tj: Sequence[int], payload) -> Matrix:
    ti = np.ascontiguousarray(ti, np.int32)
    tj = np.ascontiguousarray(tj, np.int32)
    pay = np.ascontiguousarray(payload, np.float64)
    h = _new_handle()
    _check(lib.tib_matrix_from_tiles(n, tile_size, len(ti), ti.ctypes.data_as(C.POINTER(C.c_int)),
                                     tj.ctypes.data_as(C.POINTER(C.c_int)),
                                     pay.ctypes.data_as(C.POINTER(C.c_double)), C.byref(h)))
    return Matrix(h.value)


def read_matrix_market(path: str, tile_size: int = 32) -> Matrix:
    try:
        with open(path, "rb") as f:
            text = f.read()
    except OSError:
        raise TileinvError(f"cannot open {path}") from None
    h = _new_handle()
    _check(lib.tib_matrix_read_mm(text, len(text), tile_size, C.byref(h)))
    return Matrix(h.value)


def write_matrix_market(matrix: Matrix, path: str) -> None:
    size = C.c_size_t(0)
    _check(lib.tib_matrix_write_mm(matrix._h, None, C.byref(size)))
    buf = C.create_string_buffer(size.value)
    _check(lib.tib_matrix_write_mm(matrix._h, buf, C.byref(size)))
    try:
        with open(path, "wb") as f:
            f.write(buf.raw[: size.value])
    except OSError:
        raise TileinvError(f"cannot open {path} for writing") from None


def read_matrix_tiles(path: str) -> Matrix:
    """matrix_from_tile_file(read_tile_file(path)) (tileio.cpp:55-107)."""
    h = _new_handle()
    _check(lib.tib_matrix_read_stls(path.encode(), C.byref(h)))
    return Matrix(h.value)


def read_factor_tiles(path: str, device: int = 0) -> Factor:
    """factor_from_tile_file(read_tile_file(path)): a kFactor or kPhase1 file,
    resident on `device` (the CLI's ``selinv --factor``)."""
    h = _new_handle()
    _check(lib.tib_factor_read_stls(path.encode(), device, C.byref(h)))
    return Factor(h.value)


def factor_from_tiles(n: int, tile_size: int, ti, tj, payload, phase: int = 1, device: int = 0) -> Factor:
    """A factor from host tiles: phase 1 = L (kFactor), 2 = U / W (kPhase1)."""
    ti = np.ascontiguousarray(ti, dtype=np.int32)
    tj = np.ascontiguousarray(tj, dtype=np.int32)
    pay = np.ascontiguousarray(payload, dtype=np.float64)
    h = _new_handle()
    _check(lib.tib_factor_from_tiles(n, tile_size, phase, len(ti), ti.ctypes.data_as(C.POINTER(C.c_int)),
                                     tj.ctypes.data_as(C.POINTER(C.c_int)),
                                     pay.ctypes.data_as(C.POINTER(C.c_double)), device, C.byref(h)))
    return Factor(h.value)


def factorize(matrix: Matrix, workers: int = 1, device: int = 0) -> Factor:
    """symbolic_cholesky + factorize (module.cpp:191-197)."""
    _check_workers(workers)
    h = _new_handle()
    _check(lib.tib_factorize(matrix._h, device, C.byref(h)))
    return Factor(h.value)


def selected_inverse(matrix: Matrix, selection="pattern", workers: int = 1,
                     device: int = 0) -> SelectedInverseResult:
    """selected_inverse(matrix, request, workers) (module.cpp:199-206)."""
    preset, rows, cols, ne = _request(selection)
    _check_workers(workers)
    h = _new_handle()
    _check(lib.tib_selected_inverse(matrix._h, preset, _lp(rows), _lp(cols), ne, device, C.byref(h)))
    return SelectedInverseResult(h.value)


def selected_inverse_of_factor(factor: Factor, selection="pattern",
                               workers: int = 1) -> SelectedInverseResult:
    """selected_inverse(factor, request, workers) (module.cpp:208-215)."""
    preset, rows, cols, ne = _request(selection)
    _check_workers(workers)
    h = _new_handle()
    _check(lib.tib_selected_inverse_of_factor(factor._h, preset, _lp(rows), _lp(cols), ne, C.byref(h)))
    return SelectedInverseResult(h.value)


def selected_inverse_batch(matrices: Sequence[Matrix], device: int = 0):
    """Batched factorize + pattern selected inversion of matrices sharing one
    tile pattern: returns (logdet[count], diag[count, n])."""
    count = len(matrices)
    if count == 0:
        raise TileinvError("batch needs at least one matrix")
    n = matrices[0].n
    handles = (C.c_void_p * count)(*[m._h.value for m in matrices])
    logdet = np.empty(count, np.float64)
    diag = np.empty((count, n), np.float64)
    _check(lib.tib_selected_inverse_batch(handles, count, device,
                                          logdet.ctypes.data_as(C.POINTER(C.c_double)),
                                          diag.ctypes.data_as(C.POINTER(C.c_double))))
    return logdet, diag


def factor_pattern(matrix: Matrix):
    """symbolic_fill of the matrix pattern as a list of (i, j)."""
    cnt = C.c_long()
    _check(lib.tib_symbolic_pattern(matrix._h, C.byref(cnt), None, None))
    ti = np.empty(cnt.value, np.int32)
    tj = np.empty(cnt.value, np.int32)
    _check(lib.tib_symbolic_pattern(matrix._h, C.byref(cnt), ti.ctypes.data_as(C.POINTER(C.c_int)),
                                    tj.ctypes.data_as(C.POINTER(C.c_int))))
    return list(zip(ti.tolist(), tj.tolist()))


def closure_tiles(matrix: Matrix, selection="pattern"):
    """select_tiles + symbolic_inversion closure as ((i, j) list, growth_warning)."""
    preset, rows, cols, ne = _request(selection)
    cnt, g = C.c_long(), C.c_int()
    _check(lib.tib_symbolic_closure(matrix._h, preset, _lp(rows), _lp(cols), ne, C.byref(cnt), None, None,
                                    C.byref(g)))
    ti = np.empty(cnt.value, np.int32)
    tj = np.empty(cnt.value, np.int32)
    _check(lib.tib_symbolic_closure(matrix._h, preset, _lp(rows), _lp(cols), ne, C.byref(cnt),
                                    ti.ctypes.data_as(C.POINTER(C.c_int)),
                                    tj.ctypes.data_as(C.POINTER(C.c_int)), C.byref(g)))
    return list(zip(ti.tolist(), tj.tolist())), bool(g.value)


def task_flops(matrix: Matrix, selection="pattern"):
    """Task-model FLOPs (factorize, phase1, phase2) -- SURVEY.md 8(d)."""
    preset, rows, cols, ne = _request(selection)
    f, p1, p2 = C.c_double(), C.c_double(), C.c_double()
    _check(lib.tib_flops(matrix._h, preset, _lp(rows), _lp(cols), ne, C.byref(f), C.byref(p1), C.byref(p2)))
    return f.value, p1.value, p2.value


_REPORT_KEYS = ("n_tiles", "band_b", "trsm", "trmm", "lauum", "gemm_actual", "gemm_predicted", "critical_path",
                "match")


def _report_dict(v) -> dict:
    """ComplexityReport -> dict with the reference's keys (module.cpp:109-121)."""
    out = dict(zip(_REPORT_KEYS, (int(x) for x in v)))
    out["band_b"] = None if out["band_b"] < 0 else out["band_b"]
    out["gemm_predicted"] = None if out["gemm_predicted"] < 0 else out["gemm_predicted"]
    out["match"] = bool(out["match"])
    return out


def dag_report(n_tiles: int, band: int = 0) -> dict:
    """Kernel counts and critical path of the band+arrow inversion task graph
    (count_kernels(build_band_arrow_dag(n_tiles, band or n_tiles)), module.cpp:217-223)."""
    v = (C.c_longlong * 9)()
    _check(lib.tib_dag_report(n_tiles, band, v))
    return _report_dict(v)


def dag_report_of(matrix: Matrix, selection="pattern") -> dict:
    """The same report for a matrix's filled factor pattern and the closure of
    `selection` (build_dag(symbolic_inversion(...), pattern), dag.cpp:79-190)."""
    preset, rows, cols, ne = _request(selection)
    v = (C.c_longlong * 9)()
    _check(lib.tib_dag_report_matrix(matrix._h, preset, _lp(rows), _lp(cols), ne, v))
    return _report_dict(v)


def export_dot(n_tiles: int, band: int = 0, cores: int = 0) -> str:
    """Canonical DOT text of the band+arrow task graph, nodes coloured by
    owning core when cores > 0 (module.cpp:225-233, dag.cpp:247-270)."""
    n = C.c_size_t(0)
    _check(lib.tib_dag_export_dot(n_tiles, band, cores, None, C.byref(n)))
    buf = C.create_string_buffer(n.value)
    _check(lib.tib_dag_export_dot(n_tiles, band, cores, buf, C.byref(n)))
    return buf.raw[: n.value].decode()


def predict_gemm_count(n_tiles: int, band: int) -> int:
    """Closed-form phase-2 GEMM count of the band+arrow recursion (dag.cpp:272-280)."""
    v = C.c_longlong()
    _check(lib.tib_predict_gemm_count(n_tiles, band, C.byref(v)))
    return v.value


def bench_resident(matrix: Matrix, reps: int, warmup: int, device: int = 0):
    """Device-resident timing of the fused sweep: (ms/rep, ms factor, ms phase2, logdet)."""
    a, b, c, d = C.c_double(), C.c_double(), C.c_double(), C.c_double()
    _check(lib.tib_bench_resident(matrix._h, device, reps, warmup, C.byref(a), C.byref(b), C.byref(c),
                                  C.byref(d)))
    return a.value, b.value, c.value, d.value


def device_count() -> int:
    c = C.c_int()
    _check(lib.tib_device_count(C.byref(c)))
    return c.value


__all__ = [
    "Factor", "Matrix", "NotSpdError", "SelectedInverseResult", "TileinvError", "__version__",
    "factorize", "from_dense", "from_tiles", "generate", "read_matrix_market", "selected_inverse",
    "selected_inverse_of_factor", "write_matrix_market", "selected_inverse_batch", "factor_pattern",
    "closure_tiles", "task_flops", "bench_resident", "device_count", "dag_report", "dag_report_of", "export_dot",
    "predict_gemm_count",
]


# ---- dataflow plan inspection (host only) and resident timing sessions --------

DTASK_DTYPE = np.dtype({
    "names": ["c_off", "c0_off", "cm_off", "diag_off", "p_off", "ldc", "ldc0", "m0", "n0", "seg_begin", "seg_count",
              "dep_begin", "sig_begin", "aux0", "aux1", "poll", "dep_count", "sig_count", "kind", "mode", "c_store",
              "c0_store", "cm_store", "diag_store", "dep2_count", "sig2_count"],
    "formats": ["<i8"] * 5 + ["<i4"] * 11 + ["<u2"] * 2 + ["u1"] * 8,
    "offsets": [0, 8, 16, 24, 32, 40, 44, 48, 52, 56, 60, 64, 68, 72, 76, 80, 88, 90, 92, 93, 94, 95, 96, 97, 98, 99],
    "itemsize": 104,
})
SEG_DTYPE = np.dtype({
    "names": ["a_off", "b_off", "lda", "ldb", "k_lo", "k_hi", "flags", "a_store", "b_store"],
    "formats": ["<i8", "<i8", "<i4", "<i4", "<i2", "<i2", "u1", "u1", "u1"],
    "offsets": [0, 8, 16, 20, 24, 26, 28, 29, 30],
    "itemsize": 32,
})
DEP_DTYPE = np.dtype([("counter", "<i4"), ("value", "<i4")])


def two_chain_order(matrix: Matrix):
    """(order, split) of the matrix's two-chain elimination order (order[k] =
    original tile at position k; split = first position of the second chain),
    or (None, -1) when its tile pattern admits none without fill."""
    split = C.c_int()
    order = np.zeros(matrix.n_tiles, np.int32)
    _check(lib.tib_matrix_two_chain_order(matrix._h, order.ctypes.data_as(C.POINTER(C.c_int)), C.byref(split)))
    return (order, split.value) if split.value > 0 else (None, -1)


def two_chain_permuted(matrix: Matrix) -> Matrix:
    """The matrix symmetrically permuted into its two-chain order (host tiles)."""
    h = _new_handle()
    _check(lib.tib_matrix_two_chain_permuted(matrix._h, C.byref(h)))
    return Matrix(h.value)


def plan_export(matrix: Matrix, selection="pattern", which: int = 0, crit_workers: int = 16, split: int = -1,
                batch: int = 1) -> dict:
    """Host-built dataflow plan of one device sweep (0: factorization + phase 1,
    1: phase 2 for `selection`) as numpy arrays; no GPU needed.  split > 0: the
    factor plan with a second elimination chain from that column on."""
    preset, rows, cols, ne = _request(selection)
    sizes = np.zeros(10, np.float64)
    dptr = sizes.ctypes.data_as(C.POINTER(C.c_double))
    _check(lib.tib_plan_export(matrix._h, preset, _lp(rows), _lp(cols), ne, which, crit_workers, split, batch,
                               dptr, None, None, None, None))
    nt, nq0, ns, nd, nsig, ncnt, bp, scratch, flops, tsz = sizes.tolist()
    if int(tsz) != DTASK_DTYPE.itemsize:
        raise TileinvError(f"DTask layout mismatch: {int(tsz)} vs {DTASK_DTYPE.itemsize}")
    tasks = np.zeros(int(nt), DTASK_DTYPE)
    segs = np.zeros(int(ns), SEG_DTYPE)
    deps = np.zeros(int(nd), DEP_DTYPE)
    sigs = np.zeros(int(nsig), np.int32)
    _check(lib.tib_plan_export(matrix._h, preset, _lp(rows), _lp(cols), ne, which, crit_workers, split, batch,
                               dptr, tasks.ctypes.data_as(C.c_void_p), segs.ctypes.data_as(C.c_void_p),
                               deps.ctypes.data_as(C.c_void_p), sigs.ctypes.data_as(C.c_void_p)))
    return {"tasks": tasks, "segs": segs, "deps": deps, "sigs": sigs, "q0": int(nq0), "counters": int(ncnt),
            "bp": int(bp), "scratch_doubles": int(scratch), "executed_flops": flops}


class Resident:
    """Device-resident copy of a matrix with every sweep store allocated; run()
    times `reps` fused factorize + selected-inversion sweeps with CUDA events on
    the library stream (the bench's device-side measurement)."""

    def __init__(self, matrix, device: int = 0):
        h = _new_handle()
        if isinstance(matrix, Matrix):
            _check(lib.tib_resident_create(matrix._h, device, C.byref(h)))
        else:  # a batch of matrices sharing one tile pattern
            ms = list(matrix)
            arr = (C.c_void_p * len(ms))(*[m._h.value for m in ms])
            _check(lib.tib_resident_create_batch(arr, len(ms), device, C.byref(h)))
        self._h = h

    def run(self, reps: int = 1):
        tot, f, p = C.c_double(), C.c_double(), C.c_double()
        _check(lib.tib_resident_run(self._h, reps, C.byref(tot), C.byref(f), C.byref(p)))
        return tot.value, f.value, p.value

    def info(self):
        m, e, ld, n = C.c_double(), C.c_double(), C.c_double(), C.c_long()
        _check(lib.tib_resident_info(self._h, C.byref(m), C.byref(e), C.byref(ld), C.byref(n)))
        return {"task_model_flops": m.value, "executed_flops": e.value, "logdet": ld.value,
                "kernel_launches_per_rep": n.value}

    def __del__(self, _free=lib.tib_resident_free):  # bound now: module globals are gone at interpreter exit
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            _free(h)
            self._h = None


__all__ += ["plan_export", "two_chain_order", "two_chain_permuted", "Resident", "DTASK_DTYPE", "SEG_DTYPE", "DEP_DTYPE"]
