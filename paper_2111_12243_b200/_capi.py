"""ctypes declarations of the C ABI in include/psc_b200.h.

The shared library ``libpsc_b200.so`` is built in-tree by
``__graft_entry__.build()`` (nvcc for sm_100a + g++). It is loaded lazily on
first use and there is no fallback: if the library is missing every call
raises ``LibraryMissing``.
"""
from __future__ import annotations

import ctypes as C
import os
from ctypes import POINTER, Structure, c_char_p, c_double, c_int32, c_int64, c_uint64, c_void_p

PKG_DIR = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(PKG_DIR, "libpsc_b200.so")

# status codes (psc_b200.h)
OK, ERR_INVALID_ARGUMENT, ERR_LOGIC, ERR_CUDA, ERR_NOMEM, ERR_INTERNAL = range(6)


class LibraryMissing(RuntimeError):
    pass


class CsrView(Structure):
    _fields_ = [
        ("n_rows", c_int32),
        ("n_cols", c_int32),
        ("nnz", c_int64),
        ("row_offsets", POINTER(c_int32)),
        ("col_indices", POINTER(c_int32)),
        ("values", POINTER(c_double)),
    ]


class AccessDescView(Structure):
    _fields_ = [
        ("form", c_int32),
        ("base", c_int32),
        ("stride_outer", c_int32),
        ("stride_inner", c_int32),
        ("table", POINTER(c_int32)),
        ("table_len", c_int64),
    ]


class CodeletView(Structure):
    _fields_ = [
        ("kind", c_int32),
        ("outer_extent", c_int32),
        ("inner_extent", c_int32),
        ("out", AccessDescView),
        ("mat", AccessDescView),
        ("vec", AccessDescView),
    ]


class PlanCounts(Structure):
    _fields_ = [
        ("kernel", c_int32),
        ("n_rows", c_int32),
        ("n_cols", c_int32),
        ("window", c_int32),
        ("target_groups", c_int32),
        ("nnz", c_int64),
        ("n_partitions", c_int64),
        ("n_groups", c_int64),
        ("n_codelets", c_int64),
        ("n_finalize", c_int64),
        ("n_table", c_int64),
    ]


PLAN_ARRAY_FIELDS = [
    # name, ctype, length(counts)
    ("part_group_ptr", c_int64, lambda c: c.n_partitions + 1),
    ("group_row_begin", c_int32, lambda c: c.n_groups),
    ("group_row_end", c_int32, lambda c: c.n_groups),
    ("group_strategy", c_int32, lambda c: c.n_groups),
    ("group_cost", c_int64, lambda c: c.n_groups),
    ("group_codelet_ptr", c_int64, lambda c: c.n_groups + 1),
    ("group_finalize_ptr", c_int64, lambda c: c.n_groups + 1),
    ("codelet_kind", c_int32, lambda c: c.n_codelets),
    ("codelet_m", c_int32, lambda c: c.n_codelets),
    ("codelet_n", c_int32, lambda c: c.n_codelets),
    ("desc_form", c_int32, lambda c: 3 * c.n_codelets),
    ("desc_base", c_int32, lambda c: 3 * c.n_codelets),
    ("desc_stride_outer", c_int32, lambda c: 3 * c.n_codelets),
    ("desc_stride_inner", c_int32, lambda c: 3 * c.n_codelets),
    ("desc_table_ptr", c_int64, lambda c: 3 * c.n_codelets + 1),
    ("table", c_int32, lambda c: c.n_table),
    ("fin_row", c_int32, lambda c: c.n_finalize),
    ("fin_diag_pos", c_int32, lambda c: c.n_finalize),
    ("fin_rhs_index", c_int32, lambda c: c.n_finalize),
]


class PlanArrays(Structure):
    _fields_ = [(name, POINTER(ct)) for name, ct, _ in PLAN_ARRAY_FIELDS]


class ExecContext(Structure):
    _fields_ = [
        ("matrix_values", POINTER(c_double)),
        ("gather", POINTER(c_double)),
        ("accum", POINTER(c_double)),
        ("rhs", POINTER(c_double)),
        ("solution", POINTER(c_double)),
    ]


_SIGS = {
    "psc_last_error": (c_char_p, []),
    "psc_inspect": (c_int32, [c_int32, POINTER(CsrView), c_int32, c_int32, c_int32, POINTER(c_void_p)]),
    "psc_inspect_device": (c_int32, [c_int32, POINTER(CsrView), c_int32, c_int32, c_int32, POINTER(c_void_p)]),
    "psc_plan_get_counts": (c_int32, [c_void_p, POINTER(PlanCounts)]),
    "psc_plan_to_arrays": (c_int32, [c_void_p, POINTER(CsrView), POINTER(PlanArrays)]),
    "psc_plan_from_arrays": (c_int32, [POINTER(PlanCounts), POINTER(PlanArrays), POINTER(c_void_p)]),
    "psc_plan_hash": (c_int32, [c_void_p, POINTER(CsrView), POINTER(c_uint64)]),
    "psc_plan_totals": (c_int32, [c_void_p, POINTER(c_int64), POINTER(c_int64), POINTER(c_int64)]),
    "psc_validate_plan": (c_int32, [c_void_p, POINTER(CsrView)]),
    "psc_plan_partition_rows": (c_int32, [c_void_p, c_int64, c_int64, POINTER(c_int32), POINTER(c_int32)]),
    "psc_plan_destroy": (None, [c_void_p]),
    "psc_executor_create": (c_int32, [c_int32, c_int32, POINTER(c_void_p)]),
    "psc_executor_workers": (c_int32, [c_void_p]),
    "psc_executor_set_values_version": (c_int32, [c_void_p, c_uint64]),
    "psc_executor_destroy": (None, [c_void_p]),
    "psc_bind": (c_int32, [c_void_p, c_void_p, POINTER(CsrView), c_int32, POINTER(c_void_p)]),
    "psc_bind_partitions": (
        c_int32,
        [c_void_p, c_void_p, POINTER(CsrView), c_int32, c_int64, c_int64, POINTER(c_void_p)],
    ),
    "psc_bound_rows": (c_int32, [c_void_p, POINTER(c_int32), POINTER(c_int32)]),
    "psc_bound_destroy": (None, [c_void_p]),
    "psc_bound_spmv": (c_int32, [c_void_p, c_void_p, c_void_p, c_void_p]),
    "psc_bound_sptrsv": (c_int32, [c_void_p, c_void_p, c_void_p, c_void_p, c_void_p]),
    "psc_bound_spmv_host": (c_int32, [c_void_p, POINTER(c_double), POINTER(c_double), c_void_p]),
    "psc_bound_sptrsv_host": (c_int32, [c_void_p, POINTER(c_double), POINTER(c_double), POINTER(c_double), c_void_p]),
    "psc_bound_trace": (c_int64, [c_void_p, POINTER(c_uint64), c_int64]),
    "psc_bound_launches": (c_int32, [c_void_p]),
    "psc_bound_info": (c_int32, [c_void_p, POINTER(c_int64)]),
    "psc_run_spmv": (
        c_int32,
        [c_void_p, c_void_p, POINTER(CsrView), POINTER(c_double), c_int64, POINTER(c_double), c_int64],
    ),
    "psc_run_sptrsv": (
        c_int32,
        [
            c_void_p,
            c_void_p,
            POINTER(CsrView),
            POINTER(c_double),
            c_int64,
            POINTER(c_double),
            c_int64,
            POINTER(c_double),
            c_int64,
        ],
    ),
    "psc_execute_plan": (c_int32, [c_void_p, c_void_p, POINTER(CsrView), POINTER(ExecContext)]),
    "psc_exec_blas_codelet": (c_int32, [POINTER(CodeletView), POINTER(ExecContext)]),
    "psc_exec_psci_codelet": (c_int32, [POINTER(CodeletView), POINTER(ExecContext)]),
    "psc_exec_pscii_codelet": (c_int32, [POINTER(CodeletView), POINTER(ExecContext)]),
    "psc_csr_spmv_device": (c_int32, [c_void_p, c_void_p, c_void_p, c_void_p]),
    "psc_csr_sptrsv_device": (c_int32, [c_void_p, c_void_p, c_void_p, c_void_p]),
    "psc_csr_view_of": (c_int32, [c_void_p, POINTER(CsrView)]),
    "psc_csr_destroy": (None, [c_void_p]),
    "psc_csr_from_triplets": (
        c_int32,
        [c_int32, c_int32, c_int64, POINTER(c_int32), POINTER(c_int32), POINTER(c_double), POINTER(c_void_p)],
    ),
    "psc_validate_csr": (c_int32, [POINTER(CsrView)]),
    "psc_lower_triangular": (c_int32, [POINTER(CsrView), POINTER(c_void_p)]),
    "psc_adopt_triangular": (c_int32, [POINTER(CsrView)]),
    "psc_generate_config": (c_int32, [c_int32, c_double, c_uint64, POINTER(c_void_p)]),
    "psc_seeded_vector": (None, [c_int64, c_uint64, POINTER(c_double)]),
    "psc_uniform_vector": (None, [c_int64, c_uint64, c_double, c_double, POINTER(c_double)]),
    "psc_int_vector": (None, [c_int64, c_uint64, POINTER(c_double)]),
    "psc_device_count": (c_int32, []),
    "psc_selftest_division": (c_int32, [C.c_uint64, c_int64, c_int32, C.POINTER(c_int64)]),
    "psc_bound_x_runs": (c_int32, [c_void_p, POINTER(c_int32), c_int64, POINTER(c_int64)]),
    "psc_bound_spmv_peers": (c_int32, [c_void_p, c_void_p, c_int32, c_void_p, c_void_p, c_void_p]),
    "psc_ipc_alloc": (c_int32, [c_int64, POINTER(c_void_p), C.c_char_p]),
    "psc_ipc_open": (c_int32, [C.c_char_p, POINTER(c_void_p)]),
    "psc_ipc_close": (c_int32, [c_void_p]),
    "psc_ipc_free": (c_int32, [c_void_p]),
    "psc_copy_async": (c_int32, [c_void_p, c_void_p, c_int64, c_void_p]),
    "psc_plan_save": (c_int32, [c_void_p, c_char_p]),
    "psc_csr_read_matrix_market": (c_int32, [c_char_p, POINTER(c_void_p)]),
    "psc_csr_spmv_baseline": (c_int32, [POINTER(CsrView), POINTER(c_double), c_int64, POINTER(c_double), c_int64]),
    "psc_csr_sptrsv_baseline": (c_int32, [POINTER(CsrView), POINTER(c_double), c_int64, POINTER(c_double), c_int64]),
    "psc_csr_write_matrix_market": (c_int32, [POINTER(CsrView), c_char_p]),
    "psc_plan_load": (c_int32, [c_char_p, POINTER(c_void_p)]),
}


class PeerWindow(Structure):
    """psc_peer_window (psc_b200.h)."""

    _fields_ = [("base", c_void_p), ("row_begin", c_int32), ("row_end", c_int32)]

_lib = None


def lib():
    """The loaded libpsc_b200.so (raises LibraryMissing when not built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise LibraryMissing(
                f"{LIB_PATH} is not built; run `python -c 'import __graft_entry__ as g; g.build()'`"
            )
        handle = C.CDLL(LIB_PATH, mode=C.RTLD_LOCAL)
        for name, (res, args) in _SIGS.items():
            fn = getattr(handle, name)
            fn.restype = res
            fn.argtypes = args
        _lib = handle
    return _lib


def exported_symbols():
    """Names the header declares (used by the symbol-export test)."""
    return [n for n in _SIGS]
