"""The C oracle (oracle/psc_oracle.c) -- the checker the GPU executor is held
to -- pinned against (1) the known answers of the reference's own executor
tests (test_executor.cpp), (2) golden vectors produced by the reference library
(tests/golden), and (3) the reference library itself, bitwise, on the
acceptance suite (acceptance_main.cpp:53-174) when it is built here."""
import numpy as np
import pytest

import paper_2111_12243_b200 as P
from oracle.oracle import Oracle, Ref
from paper_2111_12243_b200 import KernelKind
from paper_2111_12243_b200.psc import ExecutionContext, _codelet_view
from tests.helpers import bitwise_equal, golden_cases, suite_cases, suite_input, pattern


def _exec(which, c, ax, x, acc):
    ctx = ExecutionContext(np.array(ax, float), np.array(x, float), acc)
    v, keep = _codelet_view(c)
    Oracle.exec_codelet(which, v, ctx._c())
    return acc


def test_known_answer_codelets():
    """test_executor.cpp:37-114."""
    blas = P.Codelet(P.CodeletKind.Blas, 3, 3, P.AccessDesc.strided(0, 1, 0), P.AccessDesc.strided(0, 3, 1),
                     P.AccessDesc.strided(0, 0, 1))
    assert _exec(0, blas, range(1, 10), [1, 1, 1], np.zeros(3)).tolist() == [6, 15, 24]
    blas.vec = P.AccessDesc.strided(0, 0, 2)
    assert _exec(0, blas, range(1, 10), [1, 0, 1, 0, 1, 0], np.zeros(3)).tolist() == [6, 15, 24]
    one = P.Codelet(P.CodeletKind.Blas, 1, 1, P.AccessDesc.strided(2, 0, 0), P.AccessDesc.strided(1, 0, 1),
                    P.AccessDesc.strided(3, 0, 1))
    assert _exec(0, one, [0, 5, 0], [0, 0, 0, 4], np.ones(3)).tolist() == [1, 1, 21]
    psci = P.Codelet(P.CodeletKind.PscI, 3, 3, P.AccessDesc.strided(0, 1, 0), P.AccessDesc.strided(0, 3, 1),
                     P.AccessDesc.inner_table([0, 2, 5]))
    assert _exec(1, psci, range(1, 10), [10, 0, 20, 0, 0, 30], np.zeros(3)).tolist() == [140, 320, 500]
    p2 = P.Codelet(P.CodeletKind.PscII, 1, 2, P.AccessDesc.outer_table([0]), P.AccessDesc.strided(0, 0, 1),
                   P.AccessDesc.inner_table([1, 3]))
    assert _exec(2, p2, [2, 5], [0, 1, 0, 1], np.zeros(1)).tolist() == [7]
    f = P.Codelet(P.CodeletKind.PscII, 2, 1, P.AccessDesc.outer_table([0, 1]), P.AccessDesc.strided(0, 1, 1),
                  P.AccessDesc.point_table([1, 3]))
    assert _exec(2, f, [2, 5], [0, 1, 0, 1], np.zeros(2)).tolist() == [2, 5]


def test_known_answer_solves():
    """test_executor.cpp:148-157 (bidiagonal) and :225-241 (buffers cleared)."""
    l = P.csr_from_triplets(3, 3, [(0, 0, 2.0), (1, 0, 1.0), (1, 1, 2.0), (2, 1, 1.0), (2, 2, 2.0)])
    b = np.array([2.0, 3.0, 4.0])
    assert Oracle.sptrsv_baseline(l.view(), b).tolist() == [1, 1, 1.5]
    plan = P.inspect(KernelKind.Sptrsv, l, 2, 1)
    x, _ = Oracle.run_sptrsv(plan.export_arrays(), l.view(), b)
    assert x.tolist() == [1, 1, 1.5]
    a = pattern("dense_block(3)")
    plan = P.inspect(KernelKind.Spmv, a, 3, 1)
    assert Oracle.run_spmv(plan.export_arrays(), a.view(), np.ones(3)).tolist() == [6, 15, 24]


def test_oracle_matches_reference_golden_vectors():
    """Bitwise against outputs of the reference executor and baselines (tests/golden)."""
    for meta, a, vec, want, want_base in golden_cases():
        kk = KernelKind.Spmv if meta["kernel"] == "spmv" else KernelKind.Sptrsv
        plan = P.inspect(kk, a, meta["t"], meta["groups"])
        assert f"{plan.hash():016x}" == meta["plan_hash"], meta["name"]
        if kk == KernelKind.Spmv:
            got = Oracle.run_spmv(plan.export_arrays(), a.view(), vec)
            base = Oracle.spmv_baseline(a.view(), vec)
        else:
            got = Oracle.run_sptrsv(plan.export_arrays(), a.view(), vec)[0]
            base = Oracle.sptrsv_baseline(a.view(), vec)
        assert bitwise_equal(got, want), meta["name"]
        assert bitwise_equal(base, want_base), meta["name"]


@pytest.mark.ref
def test_oracle_matches_reference_bitwise_on_acceptance_suite():
    """Reference plan -> C oracle vs reference executor, all 336 acceptance plans."""
    n = 0
    for name, kernel, a, ints in suite_cases():
        rc = Ref.csr(a.view())
        vec = suite_input(kernel, a, ints)
        for t in (1, 2, 3, 8):
            for groups in (1, 4):
                rp = Ref.inspect(int(kernel), rc, t, groups)
                exp = rp.export()
                if kernel == KernelKind.Spmv:
                    got = Oracle.run_spmv(exp, a.view(), vec)
                    want = Ref.run_spmv(rp, rc, vec, workers=1)
                else:
                    got = Oracle.run_sptrsv(exp, a.view(), vec)[0]
                    want = Ref.run_sptrsv(rp, rc, vec, workers=1)[0]
                assert bitwise_equal(got, want), f"{name} t={t} groups={groups}"
                n += 1
    assert n == 336


@pytest.mark.ref
@pytest.mark.parametrize("config,scale", [(1, 0.04), (2, 0.03), (3, 0.002), (4, 0.01), (5, 0.001)])
def test_oracle_matches_reference_on_configs(config, scale):
    a = P.generate_config(config, scale)
    kernel = 1 if config in (2, 4) else 0
    rc = Ref.csr(a.view())
    rp = Ref.inspect(kernel, rc, 3, 8)
    vec = P.uniform_vector(a.n_cols, 10 + config)
    if kernel == 0:
        assert bitwise_equal(Oracle.run_spmv(rp.export(), a.view(), vec), Ref.run_spmv(rp, rc, vec))
    else:
        got, acc = Oracle.run_sptrsv(rp.export(), a.view(), vec)
        want, wacc = Ref.run_sptrsv(rp, rc, vec)
        assert bitwise_equal(got, want) and bitwise_equal(acc, wacc)


def test_oracle_rejects_bad_shapes():
    c = P.Codelet(P.CodeletKind.Blas, 1, 1, P.AccessDesc.strided(0, 0, 0), P.AccessDesc.strided(0, 0, 1),
                  P.AccessDesc.inner_table([0]))
    with pytest.raises(RuntimeError):
        _exec(0, c, [1], [1], np.zeros(1))
