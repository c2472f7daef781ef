"""ctypes binding of the C ABI in include/tileinv_b200.h.

The shared library is built in-tree (``paper_2504_19171_b200/libtileinv_b200.so``
by ``__graft_entry__.build()``).  There is no fallback: if the library is
missing the import fails loudly.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
# TIB_LIB_VARIANT=prof selects the profiling build (make -C csrc prof: -DTIB_PROF)
_VARIANT = os.environ.get("TIB_LIB_VARIANT", "")
LIB_PATH = os.path.join(_HERE, f"libtileinv_b200{'_' + _VARIANT if _VARIANT else ''}.so")

if not os.path.exists(LIB_PATH):
    raise ImportError(
        f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
        "(the B200 path has no CPU fallback)"
    )

lib = C.CDLL(LIB_PATH)

_i = C.c_int
_l = C.c_long
_d = C.c_double
_p = C.c_void_p
_pi = C.POINTER(C.c_int)
_pl = C.POINTER(C.c_long)
_pd = C.POINTER(C.c_double)
_pu64 = C.POINTER(C.c_uint64)
_pp = C.POINTER(C.c_void_p)

# (name, argtypes) -- every function returns int status unless noted
SIGNATURES = {
    "tib_last_not_spd": [_pl, _pi, _pi],
    "tib_device_count": [_pi],
    "tib_matrix_generate": [_l, _l, _l, _d, C.c_uint64, _i, _pp],
    "tib_matrix_generate_device": [_l, _l, _l, C.c_uint64, _i, _i, _pp],
    "tib_matrix_checksum": [_p, _pu64],
    "tib_matrix_generate_kronecker": [_i, _i, _i, _i, _d, _d, _d, _d, _d, C.c_uint64, _i, _pp],
    "tib_matrix_from_dense": [_l, _i, _pd, _pp],
    "tib_matrix_from_tiles": [_l, _i, _l, _pi, _pi, _pd, _pp],
    "tib_matrix_read_mm": [C.c_char_p, C.c_size_t, _i, _pp],
    "tib_matrix_write_mm": [_p, C.c_char_p, C.POINTER(C.c_size_t)],
    "tib_matrix_info": [_p, _pl, _pi, _pi, _pl],
    "tib_matrix_tiles": [_p, _pi, _pi, _pd],
    "tib_matrix_free": [_p],
    "tib_symbolic_pattern": [_p, _pl, _pi, _pi],
    "tib_symbolic_closure": [_p, _i, _pl, _pl, _l, _pl, _pi, _pi, _pi],
    "tib_flops": [_p, _i, _pl, _pl, _l, _pd, _pd, _pd],
    "tib_dag_report": [_i, _i, C.POINTER(C.c_longlong)],
    "tib_dag_report_matrix": [_p, _i, _pl, _pl, _l, C.POINTER(C.c_longlong)],
    "tib_dag_export_dot": [_i, _i, _i, C.c_char_p, C.POINTER(C.c_size_t)],
    "tib_predict_gemm_count": [_i, _i, C.POINTER(C.c_longlong)],
    "tib_factorize": [_p, _i, _pp],
    "tib_factor_info": [_p, _pl, _pi, _pl],
    "tib_factor_logdet": [_p, _pd],
    "tib_factor_get_tiles": [_p, _l, _pi, _pi, _pd],
    "tib_factor_replace_tiles": [_p, _l, _pi, _pi, _pd],
    "tib_factor_tiles": [_p, _i, _pi, _pi, _pd],
    "tib_factor_checksum": [_p, _pu64],
    "tib_factor_free": [_p],
    "tib_factor_phase": [_p, _pi],
    "tib_factor_from_tiles": [_l, _i, _i, _l, _pi, _pi, _pd, _i, _pp],
    "tib_factor_read_stls": [C.c_char_p, _i, _pp],
    "tib_factor_write_stls": [_p, _i, C.c_char_p],
    "tib_matrix_read_stls": [C.c_char_p, _pp],
    "tib_matrix_write_stls": [_p, C.c_char_p],
    "tib_sigma_write_stls": [_p, C.c_char_p],
    "tib_selected_inverse": [_p, _i, _pl, _pl, _l, _i, _pp],
    "tib_selected_inverse_of_factor": [_p, _i, _pl, _pl, _l, _pp],
    "tib_sigma_info": [_p, _pl, _pi, _pl, _pi],
    "tib_sigma_logdet": [_p, _pd],
    "tib_sigma_diagonal": [_p, _pd],
    "tib_sigma_entries": [_p, _pl, _pl, _pl, _pd],
    "tib_sigma_tiles": [_p, _pi, _pi, _pd],
    "tib_sigma_checksum": [_p, _pu64],
    "tib_sigma_free": [_p],
    "tib_selected_inverse_batch": [_pp, _i, _i, _pd, _pd],
    "tib_bench_resident": [_p, _i, _i, _i, _pd, _pd, _pd, _pd],
    "tib_plan_export": [_p, _i, _pl, _pl, _l, _i, _i, _i, _i, _pd, _p, _p, _p, _p],
    "tib_matrix_two_chain_order": [_p, _pi, _pi],
    "tib_matrix_two_chain_permuted": [_p, _pp],
    "tib_resident_create": [_p, _i, _pp],
    "tib_resident_create_batch": [_pp, _i, _i, _pp],
    "tib_resident_run": [_p, _i, _pd, _pd, _pd],
    "tib_resident_info": [_p, _pd, _pd, _pd, _pl],
    "tib_resident_free": [_p],
}

for _name, _args in SIGNATURES.items():
    _fn = getattr(lib, _name)
    _fn.argtypes = _args
    _fn.restype = _i

lib.tib_version.argtypes = []
lib.tib_version.restype = C.c_char_p
lib.tib_last_error_message.argtypes = []
lib.tib_last_error_message.restype = C.c_char_p

EXPORTED = sorted(list(SIGNATURES) + ["tib_version", "tib_last_error_message"])
