"""Shared test inputs: the reference acceptance suite (acceptance_main.cpp:53-82)
over the reference's own pattern matrices (tests/golden/patterns.npz, made by
tests/golden/make_golden.py with the reference generators), plus comparison
helpers."""
from __future__ import annotations

import numpy as np

import paper_2111_12243_b200 as P
from paper_2111_12243_b200 import KernelKind


def unit_lower(a: P.CsrMatrix) -> P.CsrMatrix:
    """acceptance_main.cpp:42-51 / test_helpers.hpp:16-25."""
    t = []
    for i in range(a.n_rows):
        for k in range(int(a.row_offsets[i]), int(a.row_offsets[i + 1])):
            c = int(a.col_indices[k])
            if c < i:
                t.append((i, c, float(a.values[k])))
        t.append((i, i, 1.0))
    return P.csr_from_triplets(a.n_rows, a.n_rows, t)


SUITE_SPECS = [
    ("dense_block(3)", True), ("dense_block(5)", True), ("dense_block(8)", True), ("dense_block(16)", True),
    ("banded(16,1)", True), ("banded(16,3)", True), ("banded(32,2)", True), ("banded(16,1,lower)", True),
    ("banded(32,3,lower)", True), ("scattered_gather(3,0:2:5)", True),
    ("scattered_gather(16,0:2:5:9:11:17:23:31)", True),
    ("scattered_gather(64,0:3:7:12:18:25:33:42:52:63:75:88)", True),
    ("scattered_gather(256,0:2:5:9:14:20:27:35:44:54:65:77:90:104:119:135)", True),
] + [(f"random_uniform({n},{n},{d},{s})", False) for n, d in ((16, 0.3), (64, 0.1), (128, 0.05), (256, 0.03))
     for s in (1, 7)]


_PATTERNS = None


def pattern(spec: str) -> P.CsrMatrix:
    """The reference generator's matrix for `spec` (pattern_gen.cpp), from the fixture."""
    global _PATTERNS
    if _PATTERNS is None:
        import os

        d = np.load(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "patterns.npz"))
        _PATTERNS = {}
        i = 0
        while f"p{i}_spec" in d:
            n_r, n_c = (int(v) for v in d[f"p{i}_shape"])
            _PATTERNS[d[f"p{i}_spec"].tobytes().decode()] = (n_r, n_c, d[f"p{i}_ro"], d[f"p{i}_ci"], d[f"p{i}_va"])
            i += 1
    n_r, n_c, ro, ci, va = _PATTERNS[spec]
    return P.CsrMatrix(n_r, n_c, ro.copy(), ci.copy(), va.copy())


def suite_cases():
    """42 cases: (name, kernel, matrix, integer_values) as build_suite() makes them."""
    cases = []
    for spec, ints in SUITE_SPECS:
        a = pattern(spec)
        cases.append((spec + "/solve", KernelKind.Sptrsv, unit_lower(a), ints))
        cases.append((spec, KernelKind.Spmv, a, ints))
    return cases


def suite_input(kernel, a, ints):
    """acceptance_main.cpp:137-138."""
    return P.int_vector(a.n_cols, 7) if ints else P.seeded_vector(a.n_cols, 42)


def bitwise_equal(got, want) -> bool:
    got = np.ascontiguousarray(got, dtype=np.float64)
    want = np.ascontiguousarray(want, dtype=np.float64)
    return got.shape == want.shape and np.array_equal(got.view(np.int64), want.view(np.int64))


def max_rel_err(got, want) -> float:
    """test_helpers.hpp:57-66 / bench.cpp:106-114 (elementwise, 1e-300 floor)."""
    d = np.abs(np.asarray(got) - np.asarray(want))
    mask = d != 0
    if not mask.any():
        return 0.0
    return float(np.max(d[mask] / np.maximum(np.abs(np.asarray(want)[mask]), 1e-300)))


def normwise_err(got, want) -> float:
    """max|got - want| / max|want| -- the gate SURVEY.md §8d adopts."""
    want = np.asarray(want)
    den = float(np.max(np.abs(want))) if want.size else 0.0
    num = float(np.max(np.abs(np.asarray(got) - want))) if want.size else 0.0
    return num / den if den > 0 else num


# ---- golden fixtures (tests/golden/make_golden.py, generated from the reference) ----
import json as _json  # noqa: E402
import os as _os  # noqa: E402

_GOLDEN = _os.path.join(_os.path.dirname(_os.path.abspath(__file__)), "golden")


def golden_cases():
    """[(meta, matrix, input vector, reference executor output, reference baseline output)]"""
    with open(_os.path.join(_GOLDEN, "ref_golden.json")) as f:
        index = _json.load(f)
    data = np.load(_os.path.join(_GOLDEN, "ref_golden.npz"))
    out = []
    for i, meta in enumerate(index):
        src = meta["src"]
        if src[0] == "pattern":
            a = pattern(src[1])
        elif src[0] == "pattern_unit_lower":
            a = unit_lower(pattern(src[1]))
        else:
            a = P.generate_config(int(src[1]), float(src[2]))
        if meta["input"] == "int":
            vec = P.int_vector(a.n_cols, 7)
        elif meta["input"] == "seeded":
            vec = P.seeded_vector(a.n_cols, 42)
        else:
            vec = P.uniform_vector(a.n_cols, 13, -1.0, 1.0)
        out.append((meta, a, vec, data[f"c{i}_out"], data[f"c{i}_base"]))
    return out
