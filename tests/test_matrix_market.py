"""Matrix Market ingestion (matrix_market.hpp:24-34).

The reader is checked case by case against the reference's own
read_matrix_market_file (built from its sources into oracle/_ref): the same
CSR bit for bit, or a parse error on the same 1-based line. The cases follow
test_matrix_io.cpp:60-175 (symmetric expansion, pattern and integer fields,
duplicates summed, explicit zeros kept, comments and blank lines, truncation
and malformed lines), plus the reference's data files when present."""
import os

import numpy as np
import pytest

import paper_2111_12243_b200 as P
from oracle.oracle import Ref

CASES = {
    "general_real": "%%MatrixMarket matrix coordinate real general\n3 4 4\n1 1 1.5\n2 3 -2.25\n3 4 1e-3\n3 1 7\n",
    "symmetric": "%%MatrixMarket matrix coordinate real symmetric\n3 3 4\n1 1 2\n2 1 -1\n3 2 -1\n3 3 2\n",
    "pattern_symmetric": "%%MatrixMarket matrix coordinate pattern symmetric\n3 3 3\n1 1\n3 1\n2 2\n",
    "integer": "%%MatrixMarket matrix coordinate integer general\n2 2 2\n1 2 -7\n2 1 12\n",
    "duplicates": "%%MatrixMarket matrix coordinate real general\n2 2 4\n1 1 0.1\n1 1 0.2\n2 2 1\n1 1 0.3\n",
    "explicit_zero": "%%MatrixMarket matrix coordinate real general\n2 2 2\n1 1 0\n2 2 1\n",
    "comments_blanks": ("%%MatrixMarket matrix coordinate real general\n% a comment\n\n   \n2 2 2\n% inside\n"
                        "1 1 1\n\n2 2 2\n"),
    "uppercase_header": "%%MatrixMarket MATRIX Coordinate REAL General\n1 1 1\n1 1 3\n",
    "crlf": "%%MatrixMarket matrix coordinate real general\r\n2 2 1\r\n2 1 4.5\r\n",
    "empty_matrix": "%%MatrixMarket matrix coordinate real general\n3 3 0\n",
    # errors (the reference reports the offending line)
    "empty_input": "",
    "bad_banner": "%%MatrixMarkets matrix coordinate real general\n1 1 0\n",
    "array_format": "%%MatrixMarket matrix array real general\n1 1\n1\n",
    "complex_field": "%%MatrixMarket matrix coordinate complex general\n1 1 0\n",
    "hermitian": "%%MatrixMarket matrix coordinate real hermitian\n1 1 0\n",
    "no_size_line": "%%MatrixMarket matrix coordinate real general\n% only a comment\n",
    "bad_size_line": "%%MatrixMarket matrix coordinate real general\n2 x 1\n1 1 1\n",
    "size_trailing": "%%MatrixMarket matrix coordinate real general\n2 2 1 9\n1 1 1\n",
    "symmetric_rect": "%%MatrixMarket matrix coordinate real symmetric\n2 3 1\n1 1 1\n",
    "truncated": "%%MatrixMarket matrix coordinate real general\n2 2 3\n1 1 1\n\n2 2 2\n",
    "malformed_entry": "%%MatrixMarket matrix coordinate real general\n2 2 2\n1 1 1\n2 two 2\n",
    "malformed_value": "%%MatrixMarket matrix coordinate real general\n2 2 1\n1 1 abc\n",
    "entry_trailing": "%%MatrixMarket matrix coordinate pattern general\n2 2 1\n1 1 5\n",
    "out_of_range": "%%MatrixMarket matrix coordinate real general\n2 2 2\n1 1 1\n3 1 1\n",
    "zero_index": "%%MatrixMarket matrix coordinate real general\n2 2 1\n0 1 1\n",
    "too_many": "%%MatrixMarket matrix coordinate real general\n2 2 1\n1 1 1\n2 2 2\n",
}


def _ours(path):
    try:
        return P.read_matrix_market(path), None
    except P.InvalidArgument as e:
        msg = str(e)
        assert msg.startswith("line "), msg
        return None, int(msg.split(":")[0].split()[1])


def _compare(path):
    got, got_err = _ours(path)
    ref, ref_err = Ref.read_matrix_market(path)
    if ref is None:
        assert got is None, f"reference rejects ({ref_err}), ours accepts"
        assert got_err == ref_err[0], (got_err, ref_err)
        return
    assert got is not None, f"ours rejects line {got_err}, reference accepts"
    n_rows, n_cols, ro, ci, va = ref.arrays()
    assert (got.n_rows, got.n_cols) == (n_rows, n_cols)
    assert np.array_equal(got.row_offsets, ro) and np.array_equal(got.col_indices, ci)
    assert np.array_equal(got.values.view(np.int64), va.view(np.int64))


@pytest.mark.ref
@pytest.mark.parametrize("name", sorted(CASES))
def test_reader_matches_reference(tmp_path, name):
    path = tmp_path / f"{name}.mtx"
    path.write_bytes(CASES[name].encode())
    _compare(path)


@pytest.mark.ref
def test_reference_data_files():
    data = "/root/reference/proj/tests/data"
    if not os.path.isdir(data):
        pytest.skip("reference sources not present")
    files = [f for f in sorted(os.listdir(data)) if f.endswith(".mtx")]
    assert files
    for f in files:
        _compare(os.path.join(data, f))


def test_round_trip(tmp_path):
    """write_matrix_market then read_matrix_market is the identity (17
    significant digits), on a generated matrix with awkward values."""
    a = P.generate_config(1, 0.001)
    a.values[:] = a.values * np.float64(1.0 / 3.0) + 1e-300
    path = tmp_path / "rt.mtx"
    P.write_matrix_market(a, path)
    b = P.read_matrix_market(path)
    assert b == a
    with pytest.raises(P.InvalidArgument):
        P.read_matrix_market(tmp_path / "missing.mtx")
