"""The naive CSR baselines (spmv_csr_baseline / sptrsv_csr_baseline,
/root/reference/proj/core/src/executor.cpp:310-340): the product's host
versions against the reference's golden outputs and the reference library,
and the GPU versions (psc_csr_spmv_device / psc_csr_sptrsv_device) bitwise
against the C oracle's baselines."""
import numpy as np
import pytest

import paper_2111_12243_b200 as P
from oracle.oracle import Oracle, Ref
from paper_2111_12243_b200 import KernelKind
from tests.helpers import bitwise_equal, golden_cases, pattern, unit_lower


def test_host_baselines_match_reference_golden_vectors():
    for meta, a, vec, _want, want_base in golden_cases():
        if meta["kernel"] == "spmv":
            got = P.spmv_csr_baseline(a, vec)
        else:
            got = P.sptrsv_csr_baseline(P.lower_triangular(a), vec)
        assert bitwise_equal(got, want_base), meta


@pytest.mark.ref
@pytest.mark.parametrize("spec", ["random_uniform(256,256,0.03,7)", "banded(32,3,lower)", "dense_block(16)",
                                  "scattered_gather(256,0:2:5:9:14:20:27:35:44:54:65:77:90:104:119:135)",
                                  "random_uniform(40,30,0.2,5)"])
def test_host_baselines_match_reference_library(spec):
    a = pattern(spec)
    rc = Ref.csr(a.view())
    x = P.uniform_vector(a.n_cols, 3)
    assert bitwise_equal(P.spmv_csr_baseline(a, x), Ref.spmv_baseline(rc, x))
    if a.n_rows != a.n_cols:
        return
    lo = unit_lower(a)
    rl = Ref.csr(lo.view())
    b = P.uniform_vector(lo.n_rows, 4)
    assert bitwise_equal(P.sptrsv_csr_baseline(P.TriangularMatrix.adopt(lo), b), Ref.sptrsv_baseline(rl, b))


def test_host_baselines_reject_bad_sizes():
    a = pattern("banded(32,2)")
    with pytest.raises(P.InvalidArgument):
        P.spmv_csr_baseline(a, np.zeros(a.n_cols + 1))
    lo = P.TriangularMatrix.adopt(unit_lower(a))
    with pytest.raises(P.InvalidArgument):
        P.sptrsv_csr_baseline(lo, np.zeros(a.n_rows - 1))


@pytest.mark.gpu
@pytest.mark.parametrize("config,scale", [(1, 0.05), (2, 0.1), (3, 0.01), (4, 0.02), (5, 0.005)])
def test_gpu_naive_baselines_bitwise(exe, config, scale):
    import torch

    a = P.generate_config(config, scale)
    # SpMV: one thread per row, CSR order
    plan = P.inspect(KernelKind.Spmv, a, 3, 8)
    bound = P.BoundPlan(exe, plan, a)
    x = P.uniform_vector(a.n_cols, 21)
    y = torch.full((a.n_rows,), float("nan"), dtype=torch.float64, device="cuda")
    bound.csr_spmv_naive(torch.from_numpy(x).cuda(), y)
    torch.cuda.synchronize()
    assert bitwise_equal(y.cpu().numpy(), Oracle.spmv_baseline(a.view(), x)), config
    if config == 5:  # no diagonal: no triangle to solve
        return
    lo = a if config in (2, 4) else P.lower_triangular(a).csr()
    # SpTRSV: one thread per row, sync-free
    tplan = P.inspect(KernelKind.Sptrsv, lo, 3, 8)
    tb = P.BoundPlan(exe, tplan, lo)
    b = P.uniform_vector(lo.n_rows, 22)
    xs = torch.zeros(lo.n_rows, dtype=torch.float64, device="cuda")
    for _ in range(2):  # the second call re-arms its ticket and sentinels
        tb.csr_sptrsv_naive(torch.from_numpy(b).cuda(), xs)
        torch.cuda.synchronize()
        assert bitwise_equal(xs.cpu().numpy(), Oracle.sptrsv_baseline(lo.view(), b)), config


@pytest.mark.gpu
def test_gpu_naive_sptrsv_rejects_spmv_plan(exe):
    import torch

    a = pattern("banded(32,2)")
    bound = P.BoundPlan(exe, P.inspect(KernelKind.Spmv, a, 3, 1), a)
    v = torch.zeros(a.n_rows, dtype=torch.float64, device="cuda")
    with pytest.raises(P.InvalidArgument):
        bound.csr_sptrsv_naive(v, v)
