"""Generate tests/golden/ref_golden.npz and tests/golden/patterns.npz from the
REFERENCE library (oracle/_ref/libpsc_ref.so, built from /root/reference by
oracle/Makefile).

patterns.npz holds the CSR of every reference pattern the tests use (the
acceptance suite of acceptance_main.cpp:53-82 and the golden cases below),
made by the reference's own generators (pattern_gen.cpp) -- the product has
no copy of them.

For every case: the reference inspector's plan digest (include/psc_plan_hash.h),
total cost / ops, and the outputs of the reference executor (run_spmv /
run_sptrsv, workers=1) and of the reference naive baselines, on seeded inputs.
Config matrices are rebuilt at test time from configs.cpp (compiled into both
libraries), so only digests and vectors are stored for them. Run in the build container:  python tests/golden/make_golden.py
"""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import paper_2111_12243_b200 as P  # noqa: E402
from oracle.oracle import Ref  # noqa: E402
from tests.helpers import SUITE_SPECS, pattern, unit_lower  # noqa: E402

EXTRA_SPECS = ["dense_block(3)", "dense_block(7)", "banded(20,3)", "banded(20,2,lower)", "scattered_gather(5,9:0:3:3)",
               "random_uniform(40,30,0.2,5)", "random_uniform(200,200,0.04,3)", "random_uniform(64,64,0.1,9)",
               "dense_block(2)", "dense_block(4)", "dense_block(6)", "scattered_gather(3,0:2:5)",
               "scattered_gather(6,0:1:2:3)", "banded(4,0,lower)", "banded(4,1,lower)",
               "random_uniform(30,30,0.2,17)"]

CASES = [
    # (name, matrix source, kernel, t, groups, input kind)
    ("dense_block(8)", ("pattern", "dense_block(8)"), "spmv", 3, 1, "int"),
    ("dense_block(8)/solve", ("pattern_unit_lower", "dense_block(8)"), "sptrsv", 3, 1, "int"),
    ("banded(32,2)", ("pattern", "banded(32,2)"), "spmv", 2, 4, "int"),
    ("banded(32,3,lower)/solve", ("pattern_unit_lower", "banded(32,3,lower)"), "sptrsv", 3, 4, "int"),
    ("scattered_gather(64)", ("pattern", "scattered_gather(64,0:3:7:12:18:25:33:42:52:63:75:88)"), "spmv", 8, 4, "int"),
    ("random_uniform(128,7)", ("pattern", "random_uniform(128,128,0.05,7)"), "spmv", 3, 4, "seeded"),
    ("random_uniform(128,7)/solve", ("pattern_unit_lower", "random_uniform(128,128,0.05,7)"), "sptrsv", 3, 4,
     "seeded"),
    ("random_uniform(256,1)", ("pattern", "random_uniform(256,256,0.03,1)"), "spmv", 1, 1, "seeded"),
    ("config1@30^2", ("config", 1, 0.0009), "spmv", 3, 8, "uniform"),
    ("config2@10^3", ("config", 2, 0.001), "sptrsv", 3, 8, "uniform"),
    ("config3@4^3", ("config", 3, 0.000125), "spmv", 3, 8, "uniform"),
    ("config4@800", ("config", 4, 0.002), "sptrsv", 3, 8, "uniform"),
    ("config5@400", ("config", 5, 0.00002), "spmv", 3, 8, "uniform"),
]


def write_patterns():
    specs = [s for s, _ in SUITE_SPECS] + EXTRA_SPECS + [c[1][1] for c in CASES if c[1][0] != "config"]
    out = {}
    for i, spec in enumerate(dict.fromkeys(specs)):
        n_r, n_c, ro, ci, va = Ref.generate_pattern(spec).arrays()
        out[f"p{i}_shape"] = np.array([n_r, n_c], dtype=np.int64)
        out[f"p{i}_ro"], out[f"p{i}_ci"], out[f"p{i}_va"] = ro, ci, va
        out[f"p{i}_spec"] = np.frombuffer(spec.encode(), dtype=np.uint8)
    np.savez_compressed(os.path.join(os.path.dirname(__file__), "patterns.npz"), **out)


def build(src):
    if src[0] == "pattern":
        return pattern(src[1])
    if src[0] == "pattern_unit_lower":
        return unit_lower(pattern(src[1]))
    return P.generate_config(src[1], src[2])


def make_input(kind, n):
    if kind == "int":
        return P.int_vector(n, 7)
    if kind == "seeded":
        return P.seeded_vector(n, 42)
    return P.uniform_vector(n, 13, -1.0, 1.0)


def main():
    assert Ref.available(), "the reference library must be built (make -C oracle ref)"
    write_patterns()
    out, index = {}, []
    for i, (name, src, kernel, t, groups, kind) in enumerate(CASES):
        a = build(src)
        rc = Ref.csr(a.view())
        k = 0 if kernel == "spmv" else 1
        plan = Ref.inspect(k, rc, t, groups)
        vec = make_input(kind, a.n_cols)
        if kernel == "spmv":
            y = Ref.run_spmv(plan, rc, vec)
            base = Ref.spmv_baseline(rc, vec)
        else:
            y, _acc = Ref.run_sptrsv(plan, rc, vec)
            base = Ref.sptrsv_baseline(rc, vec)
        cost, ops = plan.totals()
        out[f"c{i}_out"] = y
        out[f"c{i}_base"] = base
        index.append({"name": name, "src": list(src), "kernel": kernel, "t": t, "groups": groups, "input": kind,
                      "n_rows": a.n_rows, "nnz": a.nnz(), "plan_hash": f"{plan.hash():016x}", "total_cost": cost,
                      "total_ops": ops})
    np.savez_compressed(os.path.join(os.path.dirname(__file__), "ref_golden.npz"), **out)
    with open(os.path.join(os.path.dirname(__file__), "ref_golden.json"), "w") as f:
        json.dump(index, f, indent=1)
    print(f"wrote {len(index)} cases")


if __name__ == "__main__":
    main()
