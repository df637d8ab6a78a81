"""Fast mode (PSC_MODE_FAST, spmv_fast.cu) against the reference's naive
baseline, as computed by the C oracle (oracle/psc_oracle.c, pinned to the
reference in test_oracle.py).

Bar (north_star): SpMV within 1e-12 normwise of the reference (the summation
order differs); exact on integer data whose sums stay below 2^53;
deterministic run to run; and the placeholder entries of rows that are empty
in a column pass contribute nothing, even when x holds NaN or Inf."""
import os

import numpy as np
import pytest

import paper_2111_12243_b200 as P
from oracle.oracle import Oracle
from paper_2111_12243_b200 import KernelKind
from tests.helpers import normwise_err, pattern, suite_cases, suite_input

pytestmark = pytest.mark.gpu
FAST = 1


def fast_bound(exe, a, split_bytes=None, per=None):
    env = {}
    if split_bytes is not None:
        env["PSC_FAST_SPLIT_BYTES"] = str(split_bytes)
    if per is not None:
        env["PSC_FAST_PER"] = str(per)
    old = {k: os.environ.get(k) for k in env}
    os.environ.update(env)
    try:
        plan = P.inspect(KernelKind.Spmv, a, 3, 8)
        return P.BoundPlan(exe, plan, a, mode=FAST), plan
    finally:
        for k, v in old.items():
            if v is None:
                del os.environ[k]
            else:
                os.environ[k] = v


def multiply(b, x, host=False):
    import torch

    if host:
        y = np.full(b.row_end - b.row_begin, np.nan)
        b.spmv_host(np.ascontiguousarray(x), y)
        torch.cuda.synchronize()
        return y
    xd = torch.from_numpy(np.ascontiguousarray(x)).cuda()
    yd = torch.full((max(1, b.row_end - b.row_begin),), float("nan"), dtype=torch.float64, device="cuda")
    b.spmv(xd, yd)
    torch.cuda.synchronize()
    return yd.cpu().numpy()[: b.row_end - b.row_begin]


def test_acceptance_suite_fast(exe):
    """Every SpMV matrix of the acceptance suite (acceptance_main.cpp:53-82):
    within 1e-12 normwise of the naive baseline, exact on integer data."""
    n_fast = 0
    for name, kernel, a, ints in suite_cases():
        if kernel != KernelKind.Spmv:
            continue
        x = suite_input(kernel, a, ints)
        want = Oracle.spmv_baseline(a.view(), x)
        for per in (4, 8):
            b, _ = fast_bound(exe, a, split_bytes=-1, per=per)  # (set: the entry streams even for short rows)
            got = multiply(b, x)
            n_fast += b.info()["path"] == 2
            if ints:
                assert np.array_equal(got, want), name
            else:
                assert normwise_err(got, want) <= 1e-12, name
    assert n_fast > 0


@pytest.mark.parametrize("config,scale", [(1, 1.0), (1, 0.01), (5, 0.02), (5, 0.2)])
def test_configs_fast(exe, config, scale):
    """Config 5: the flagged entry streams; config 1 (rows of <= 16 entries, one
    pass): the thread-per-row kernel, which is faster there and bitwise the
    parity result."""
    a = P.generate_config(config, scale)
    x = P.uniform_vector(a.n_cols, 10 + config)
    b, plan = fast_bound(exe, a)
    assert b.info()["path"] == (0 if config == 1 else 2)
    if config == 1:
        assert np.array_equal(multiply(b, x).view(np.int64),
                              Oracle.run_spmv(plan.export_arrays(), a.view(), x).view(np.int64))
    got = multiply(b, x)
    assert normwise_err(got, Oracle.spmv_baseline(a.view(), x)) <= 1e-12
    assert np.array_equal(got.view(np.int64), multiply(b, x).view(np.int64))  # deterministic
    assert np.array_equal(got.view(np.int64), multiply(b, x, host=True).view(np.int64))  # host path (y slices)


@pytest.mark.parametrize("split_bytes", [-1, 16000, 4000])
def test_fast_column_passes_and_host_path(exe, split_bytes):
    """Forced column passes (4 ranges, the most, at n = 4000 columns), on the
    device and through the host-buffer path."""
    a = P.generate_config(5, 0.0002)
    x = P.uniform_vector(a.n_cols, 15)
    want = Oracle.spmv_baseline(a.view(), x)
    b, _ = fast_bound(exe, a, split_bytes=split_bytes)
    assert b.info()["passes_or_block_rows"] == (1 if split_bytes < 0 else min(4, -(-8 * a.n_cols // split_bytes)))
    got = multiply(b, x)
    assert normwise_err(got, want) <= 1e-12
    assert np.array_equal(multiply(b, x, host=True).view(np.int64), got.view(np.int64))


def rows_matrix(lengths, n_cols, seed=3):
    rng = np.random.default_rng(seed)
    ro = np.zeros(len(lengths) + 1, dtype=np.int64)
    ro[1:] = np.cumsum(lengths)
    ci = np.concatenate([np.sort(rng.choice(n_cols, size=l, replace=False)) for l in lengths]) if sum(lengths) else \
        np.zeros(0, np.int32)
    va = rng.uniform(-1, 1, int(ro[-1]))
    return P.CsrMatrix(len(lengths), n_cols, ro, ci, va)


@pytest.mark.parametrize("lengths,n_cols", [
    ([0, 0, 5, 0, 3, 0, 0], 16),                  # empty rows first, between and last
    ([0] * 50, 10),                                # no entries at all
    ([7], 9),                                      # one row
    ([3000, 1, 0, 2500, 4, 0, 0, 6000], 9000),     # rows spanning many 128/256-entry chunks
    ([1] * 700 + [300] + [2] * 700, 2000),         # chunk boundaries inside and between rows
    ([5, 0, 9] * 300, 50),                         # rectangular, more rows than columns
])
def test_fast_ragged_rows(exe, lengths, n_cols):
    a = rows_matrix(lengths, n_cols)
    x = P.uniform_vector(a.n_cols, 21)
    want = Oracle.spmv_baseline(a.view(), x)
    for split in (-1, max(8, 8 * n_cols // 3)):
        b, _ = fast_bound(exe, a, split_bytes=split)
        got = multiply(b, x)
        assert normwise_err(got, want) <= 1e-12
        # the host path runs the last pass in row slices cut where no carry crosses: same sums
        assert np.array_equal(multiply(b, x, host=True).view(np.int64), got.view(np.int64))


def test_fast_placeholders_do_not_touch_x(exe):
    """A row empty in a column pass holds a placeholder entry: it must add +0
    without reading x, so NaN / Inf in x reach only the rows that use them."""
    a = rows_matrix([0, 2, 0, 3, 0], 6, seed=9)
    x = P.uniform_vector(6, 4)
    x[0] = np.nan
    x[5] = np.inf
    want = Oracle.spmv_baseline(a.view(), x)
    for split in (-1, 16):
        b, _ = fast_bound(exe, a, split_bytes=split)
        got = multiply(b, x)
        assert np.array_equal(multiply(b, x, host=True).view(np.int64), got.view(np.int64))
        assert np.array_equal(np.isnan(got), np.isnan(want))
        fin = np.isfinite(want)
        assert np.array_equal(got[~fin & ~np.isnan(want)], want[~fin & ~np.isnan(want)])  # the infinities
        assert normwise_err(got[fin], want[fin]) <= 1e-12


def test_fast_mode_falls_back_to_parity_for_segmented_plans(exe):
    """Fast mode changes only single-segment-row SpMV plans; a segmented plan
    (BLAS tiles) and the solve keep the bitwise parity kernels."""
    a = pattern("dense_block(16)")
    x = P.int_vector(a.n_cols, 7)
    b, plan = fast_bound(exe, a)
    if b.info()["path"] != 2:
        assert np.array_equal(multiply(b, x), Oracle.run_spmv(plan.export_arrays(), a.view(), x))
