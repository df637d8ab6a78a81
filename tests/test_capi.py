"""The C-ABI library: loads, exports every symbol include/psc_b200.h declares,
maps errors onto the reference's exception types, and its matrix helpers
reproduce the reference's (csr_from_triplets, lower_triangular, the seeded
vector streams). The reference's pattern generators are not in the product:
the tests take their matrices from tests/golden/patterns.npz."""
import os
import re

import ctypes as C

import numpy as np
import pytest

import paper_2111_12243_b200 as P
from oracle.oracle import Ref, RefCsr
from paper_2111_12243_b200 import _capi
from tests.helpers import SUITE_SPECS, pattern

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    text = open(os.path.join(ROOT, "include", "psc_b200.h")).read()
    return sorted(set(re.findall(r"PSC_API[^;(]*?\b(psc_\w+)\s*\(", text, flags=re.S)))


def test_library_exports_every_declared_symbol():
    lib = _capi.lib()
    names = header_symbols()
    assert len(names) >= 40
    for n in names:
        assert hasattr(lib, n), n
    exported = os.popen(f"nm -D --defined-only {_capi.LIB_PATH}").read()
    for n in names:
        assert re.search(rf"\b{n}\b", exported), n


def test_sm100a_code_is_in_the_library():
    out = os.popen(f"cuobjdump --list-elf {_capi.LIB_PATH} 2>/dev/null").read()
    assert "sm_100a" in out


def test_executor_argument_errors():
    """executor.cpp:253-255 (workers < 1 -> invalid_argument)."""
    with pytest.raises(P.InvalidArgument):
        P.Executor(0)
    if P.device_count() == 0:
        with pytest.raises(P.CudaError):
            P.Executor(1)


def test_csr_helpers():
    a = P.csr_from_triplets(2, 3, [(1, 2, 1.0), (0, 1, 2.0), (1, 2, 3.0), (1, 0, 4.0)])
    assert a.row_offsets.tolist() == [0, 1, 3]
    assert a.col_indices.tolist() == [1, 0, 2]
    assert a.values.tolist() == [2.0, 4.0, 4.0]
    with pytest.raises(P.InvalidArgument):
        P.csr_from_triplets(2, 2, [(2, 0, 1.0)])
    with pytest.raises(P.InvalidArgument):
        P.lower_triangular(P.csr_from_triplets(2, 3, [(0, 0, 1.0)]))
    with pytest.raises(P.InvalidArgument):  # missing diagonal
        P.lower_triangular(P.csr_from_triplets(2, 2, [(0, 0, 1.0), (1, 0, 1.0)]))
    l = P.lower_triangular(pattern("dense_block(3)"))
    assert l.csr().nnz() == 6 and l.diag_pos(2) == 5
    bad = P.CsrMatrix(2, 2, [0, 2, 3], [1, 0, 1], [1.0, 1.0, 1.0])
    with pytest.raises(P.InvalidArgument):
        P.validate_csr(bad)


@pytest.mark.ref
def test_csr_from_triplets_matches_the_reference():
    """csr_matrix.cpp:9-45: unsorted triplets with duplicates (summed in input order)."""
    rng = np.random.default_rng(5)
    for n_rows, n_cols, n in [(1, 1, 0), (7, 5, 60), (40, 33, 900), (3, 1000, 50)]:
        r = rng.integers(0, n_rows, n).astype(np.int32)
        c = rng.integers(0, n_cols, n).astype(np.int32)
        v = rng.uniform(-1, 1, n) * 10.0 ** rng.integers(-8, 8, n)
        mine = P.csr_from_triplets(n_rows, n_cols, list(zip(r.tolist(), c.tolist(), v.tolist())))
        h = C.c_void_p()
        Ref._check(Ref.lib().ref_csr_from_triplets(n_rows, n_cols, n, r.ctypes.data_as(C.POINTER(C.c_int32)),
                                                   c.ctypes.data_as(C.POINTER(C.c_int32)),
                                                   v.ctypes.data_as(C.POINTER(C.c_double)), C.byref(h)))
        _, _, ro, ci, va = RefCsr(h).arrays()
        assert np.array_equal(mine.row_offsets, ro) and np.array_equal(mine.col_indices, ci)
        assert np.array_equal(mine.values.view(np.int64), va.view(np.int64))


@pytest.mark.ref
def test_pattern_fixtures_are_the_reference_generators():
    for spec, _ in SUITE_SPECS:
        mine = pattern(spec)
        n_r, n_c, ro, ci, va = Ref.generate_pattern(spec).arrays()
        assert (mine.n_rows, mine.n_cols) == (n_r, n_c)
        assert np.array_equal(mine.row_offsets, ro) and np.array_equal(mine.col_indices, ci)
        assert np.array_equal(mine.values, va)
    assert np.array_equal(P.int_vector(50, 3), Ref.int_vector(50, 3))


@pytest.mark.ref
def test_reference_arm_inputs_equal_the_products():
    """bench.py's reference arm generates its inputs inside the reference library
    (configs.cpp compiled in by oracle/Makefile); they must be the product's."""
    for config, scale in [(1, 0.01), (2, 0.001), (3, 0.000125), (4, 0.002), (5, 0.0001)]:
        mine = P.generate_config(config, scale)
        n_r, n_c, ro, ci, va = Ref.generate_config(config, scale).arrays()
        assert (mine.n_rows, mine.n_cols) == (n_r, n_c)
        assert np.array_equal(mine.row_offsets, ro) and np.array_equal(mine.col_indices, ci)
        assert np.array_equal(mine.values.view(np.int64), va.view(np.int64))
    assert np.array_equal(P.uniform_vector(1000, 15), Ref.uniform_vector(1000, 15))


def test_config_generators_shapes():
    """BASELINE.json shapes at small scale (DESIGN.md Inputs)."""
    c1 = P.generate_config(1, 0.01)  # N = 100
    assert c1.n_rows == 10000 and c1.nnz() == 5 * 10000 - 4 * 100
    c2 = P.generate_config(2, 0.001)  # N = 10
    assert c2.n_rows == 1000 and c2.nnz() == 4 * 1000 - 3 * 100
    P.TriangularMatrix.adopt(c2)
    c3 = P.generate_config(3, 0.000125)  # N = 4
    assert c3.n_rows == 192 and c3.nnz() == 9 * (3 * 4 - 2) ** 3
    c4 = P.generate_config(4, 0.002)
    P.TriangularMatrix.adopt(c4)
    c5 = P.generate_config(5, 0.0001)
    assert c5.n_rows == 2000
    assert np.array_equal(c5.col_indices, P.generate_config(5, 0.0001).col_indices)  # deterministic
    # symmetric pattern
    dense = np.zeros((2000, 2000))
    for r in range(2000):
        dense[r, c5.col_indices[c5.row_offsets[r]:c5.row_offsets[r + 1]]] = 1
    assert np.array_equal(dense, dense.T)
