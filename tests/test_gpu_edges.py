"""GPU edge cases for every kernel path, bitwise against the C oracle
(oracle/psc_oracle.c, pinned to the reference in test_oracle.py): empty and
tiny matrices, empty rows, rectangular shapes, the boundaries between kernel
variants (thread-per-row <= 16 entries vs warp chunks; warp chunks <= 256 vs
long rows; record rounds <= 4 off-diagonal entries vs the unit queue; queue
rows <= 2048 entries vs its per-lane path), single chains and dense
triangles."""
import numpy as np
import pytest

import paper_2111_12243_b200 as P
from oracle.oracle import Oracle
from paper_2111_12243_b200 import KernelKind
from tests.helpers import bitwise_equal

pytestmark = pytest.mark.gpu


def _csr(n_rows, n_cols, entries):
    return P.csr_from_triplets(n_rows, n_cols, entries)


def _lower(n, row_cols, seed=0):
    """Lower triangle: row r has the given off-diagonal columns and a
    dominant diagonal (stored last)."""
    rng = np.random.default_rng(seed)
    ent = []
    for r in range(n):
        cs = sorted(set(int(c) for c in row_cols(r) if 0 <= c < r))
        for c in cs:
            ent.append((r, c, float(rng.uniform(-1, 1))))
        ent.append((r, r, float(2 + len(cs) + rng.uniform(0, 1))))
    return _csr(n, n, ent)


def _spmv_check(exe, a, seed=3):
    plan = P.inspect(KernelKind.Spmv, a, 3, 8)
    x = P.uniform_vector(a.n_cols, seed)
    y = np.full(a.n_rows, np.nan)
    P.run_spmv(plan, a, x, y, exe)
    assert bitwise_equal(y, Oracle.run_spmv(plan.export_arrays(), a.view(), x))


def _sptrsv_check(exe, a, seed=4):
    plan = P.inspect(KernelKind.Sptrsv, a, 3, 8)
    b = P.uniform_vector(a.n_rows, seed)
    x = np.full(a.n_rows, np.nan)
    acc = np.full(a.n_rows, np.nan)
    P.run_sptrsv(plan, P.TriangularMatrix.adopt(a), b, x, acc, exe)
    want, want_acc = Oracle.run_sptrsv(plan.export_arrays(), a.view(), b)[:2]
    assert bitwise_equal(x, want)
    assert bitwise_equal(acc, want_acc)


def test_spmv_tiny_and_empty(exe):
    _spmv_check(exe, _csr(1, 1, [(0, 0, 2.5)]))
    _spmv_check(exe, _csr(5, 3, [(0, 2, 1.0), (4, 0, -2.0)]))  # empty rows, rectangular
    _spmv_check(exe, _csr(3, 7, [(1, c, 0.5 * c) for c in range(7)]))
    a = _csr(4, 4, [])
    plan = P.inspect(KernelKind.Spmv, a, 3, 8)
    y = np.full(4, np.nan)
    P.run_spmv(plan, a, np.ones(4), y, exe)
    assert np.array_equal(y, np.zeros(4))


@pytest.mark.parametrize("width", [1, 4, 5, 16, 17, 255, 256, 257, 5000])
def test_spmv_row_length_boundaries(exe, width):
    """Rows of exactly `width` entries (plus a short row), across the
    thread-per-row / chunk / long-row boundaries."""
    n = 300
    rng = np.random.default_rng(width)
    ent = []
    for r in range(n):
        w = width if r % 3 else 2
        cols = rng.choice(6000, size=min(w, 6000), replace=False)
        ent += [(r, int(c), float(rng.uniform(-1, 1))) for c in cols]
    _spmv_check(exe, _csr(n, 6000, ent))


@pytest.mark.parametrize("width", [1, 3, 4, 5, 7, 8, 9, 12, 13, 16])
def test_spmv_shifted_runs(monkeypatch, width):
    """Banded matrices of short rows: interior rows form shifted runs (the
    same length, the columns of the row above plus one) and take
    spmv_run_kernel's template path (no row offsets or column loads); rows
    clipped by the matrix edge, rows that break a run, runs shorter than the
    minimum, empty rows and a wide rectangular tail go through CSR in the same
    kernel. Bitwise equal to the oracle through run_spmv and through the
    bound device path, and to the row kernel (PSC_SPMV_RUNS=0)."""
    import torch
    n, n_cols = 1500, 1700
    rng = np.random.default_rng(100 + width)
    offs = sorted(set([0, 1, -1, 40, -40, 3, -3, 100, -7, 11, 23, -100, 57, -57, 150, 170][:width]))
    ent = []
    for r in range(n):
        if 200 <= r < 215:
            continue  # empty rows
        if r % 97 == 5 or 300 <= r < 330 and r % 2:  # rows that break runs; runs of one row
            cols = rng.choice(n_cols, size=rng.integers(1, min(16, width + 2) + 1), replace=False)
        else:
            cols = [r + o for o in offs if 0 <= r + o < n_cols]
        ent += [(r, int(c), float(rng.uniform(-1, 1))) for c in cols]
    a = _csr(n, n_cols, ent)
    plan = P.inspect(KernelKind.Spmv, a, 3, 8)
    x = P.uniform_vector(a.n_cols, 7)
    want = Oracle.run_spmv(plan.export_arrays(), a.view(), x)
    units = {}
    for runs in ("1", "0"):
        monkeypatch.setenv("PSC_SPMV_RUNS", runs)
        exe = P.Executor(1)
        y = np.full(a.n_rows, np.nan)
        P.run_spmv(plan, a, x, y, exe)
        assert bitwise_equal(y, want), (width, runs)
        for mode in (0, 1):  # PSC_MODE_PARITY, PSC_MODE_FAST: one-pass short-row plans share the kernel
            bound = P.BoundPlan(exe, plan, a, mode=mode)
            yd = torch.full((a.n_rows,), float("nan"), dtype=torch.float64, device="cuda")
            bound.spmv(torch.from_numpy(x).cuda(), yd)
            assert bitwise_equal(yd.cpu().numpy(), want), (width, runs, mode)
            units[runs] = bound.info()["work_units"]
    assert units["1"] != units["0"]  # the run items were in use


def test_sptrsv_tiny(exe):
    _sptrsv_check(exe, _csr(1, 1, [(0, 0, 3.0)]))
    _sptrsv_check(exe, _lower(50, lambda r: []))  # diagonal only
    _sptrsv_check(exe, _lower(2, lambda r: [r - 1]))


def test_sptrsv_single_long_chain(exe):
    _sptrsv_check(exe, _lower(20000, lambda r: [r - 1]))


def test_sptrsv_dense_triangle(exe):
    """A dense 300 x 300 triangle: rows up to 299 entries (unit queue)."""
    _sptrsv_check(exe, _lower(300, lambda r: range(r)))


@pytest.mark.parametrize("stream", ["1", "0"])
def test_sptrsv_row_longer_than_queue_buffer(monkeypatch, stream):
    """One row with 2500 off-diagonal entries (> the queue kernel's
    2048-entry product buffer: its per-lane path; > the streaming kernel's
    staged row tail)."""
    monkeypatch.setenv("PSC_TRSV_STREAM", stream)
    exe = P.Executor(1)
    _sptrsv_check(exe, _lower(2600, lambda r: range(r) if r == 2599 else ([r - 1] if r else [])))


@pytest.mark.parametrize("stream", ["1", "0"])
def test_sptrsv_mixed_short_and_long_rows(monkeypatch, stream):
    """Mostly stencil-like rows with a few wide rows: the plan is not
    record-eligible as a whole, so the whole solve takes the long-row path:
    the lane-per-row streaming kernel (chain mode) or the warp-per-row unit
    queue (PSC_TRSV_STREAM=0)."""
    monkeypatch.setenv("PSC_TRSV_STREAM", stream)
    exe = P.Executor(1)
    _sptrsv_check(exe, _lower(3000, lambda r: [r - 1, r - 40, r - 900] if r % 97 else range(max(0, r - 60), r)))
    # supernode-like dense triangles longer than a 32-row piece, with dense runs over earlier ones
    def rows(r):
        s0 = (r // 45) * 45
        prev = list(range(max(0, s0 - 45), s0)) if r % 3 else []
        return prev + list(range(s0, r))
    _sptrsv_check(exe, _lower(1000, rows))


@pytest.mark.parametrize("lean", ["2", "4"])
def test_sptrsv_kernels_on_chain_and_stencil(monkeypatch, lean):
    monkeypatch.setenv("PSC_TRSV_LEAN", lean)
    exe = P.Executor(1)
    _sptrsv_check(exe, _lower(4000, lambda r: [r - 1, r - 63, r - 64 * 64]))
    _sptrsv_check(exe, _lower(500, lambda r: [r - 2, r - 7]))  # no chains (row mode)


@pytest.mark.parametrize("with_acc", [True, False])
def test_sptrsv_division_fallback(exe, with_acc):
    """Diagonals and right-hand sides far outside the exponent range of the
    reciprocal-based division ([-500, 500]): the record kernel's rare
    __ddiv_rn fallback (for t = b - acc and for the diagonal, flagged at pack
    time), with and without the acc output (separate kernel instantiations),
    bitwise against the oracle."""
    import torch

    n = 3000
    rng = np.random.default_rng(11)
    ent = []
    for r in range(n):
        cs = [c for c in (r - 1, r - 40, r - 900) if c >= 0]
        for c in cs:
            ent.append((r, c, float(rng.uniform(-1, 1))))
        d = 2.0 + len(cs)
        if r % 7 == 3:
            d *= 1e-160  # tiny diagonal: flagged at pack time
        elif r % 11 == 5:
            d *= 1e170  # huge diagonal
        ent.append((r, r, d))
    a = _csr(n, n, ent)
    plan = P.inspect(KernelKind.Sptrsv, a, 3, 8)
    b = P.uniform_vector(n, 12)
    b[::13] *= 1e-300  # tiny and subnormal-range right-hand sides
    b[5::17] *= 1e200
    want, want_acc = Oracle.run_sptrsv(plan.export_arrays(), a.view(), b)[:2]
    bound = P.BoundPlan(exe, plan, a)
    bd = torch.from_numpy(b).cuda()
    xd = torch.full_like(bd, float("nan"))
    if with_acc:
        accd = torch.full_like(bd, float("nan"))
        bound.sptrsv(bd, xd, accd)
    else:
        bound.sptrsv(bd, xd)
    torch.cuda.synchronize()
    assert bitwise_equal(xd.cpu().numpy(), want)
    if with_acc:
        assert bitwise_equal(accd.cpu().numpy(), want_acc)


def _block_rows_matrix(seed=21):
    """Dense dof blocks over stencil-like neighbour runs: nodes 0..299 with
    2, 3 or 4 dof (by thirds), neighbours i-1..i+1 and i+-10 (separate x
    runs); every 50th node reads i-30..i+30 (> 96 entries per row)."""
    rng = np.random.default_rng(seed)
    n_nodes = 300
    dof = np.array([2 if i < 100 else (3 if i < 200 else 4) for i in range(n_nodes)])
    start = np.concatenate([[0], np.cumsum(dof)])
    ent = []
    for i in range(n_nodes):
        if i % 50 == 7:
            nbrs = range(max(0, i - 30), min(n_nodes, i + 31))
        else:
            nbrs = [j for j in (i - 10, i - 1, i, i + 1, i + 10) if 0 <= j < n_nodes]
        for d in range(dof[i]):
            for j in nbrs:
                for e in range(dof[j]):
                    ent.append((int(start[i] + d), int(start[j] + e), float(rng.uniform(-1, 1))))
    n = int(start[-1])
    return _csr(n, n, ent)


@pytest.mark.parametrize("groups", ["1", "0"])
def test_spmv_row_groups(monkeypatch, groups):
    """Rows of a node share one BLAS segment template: with groups on they
    form row groups of 2 or 3 rows (a 4-dof node splits 3 + 1), wide rows
    and boundary rows stay in chunks. Bitwise against the oracle, with and
    without groups."""
    monkeypatch.setenv("PSC_SPMV_GROUPS", groups)
    exe = P.Executor(1)
    _spmv_check(exe, _block_rows_matrix())


@pytest.mark.parametrize("force,parts", [(True, "2"), (True, "3"), (True, "4"), (False, "2")])
def test_spmv_column_split(monkeypatch, force, parts):
    """Column-split passes (the matrix as two CSRs by column half, the rows'
    dot_unit state carried between the passes; 2, 3 or 4 column ranges): power-law rows with long
    rows, empty rows, rows entirely in one half, and rows whose lane sums /
    tail straddle the split. Bitwise against the oracle with the split forced
    on (PSC_SPMV_SPLIT_BYTES=1) and off."""
    import torch

    monkeypatch.setenv("PSC_SPMV_SPLIT_BYTES", "1" if force else "-1")
    monkeypatch.setenv("PSC_SPMV_SPLIT_PARTS", parts)
    exe = P.Executor(1)
    rng = np.random.default_rng(31)
    n = 3000
    ent = []
    for r in range(n):
        k = int(min(2000, rng.zipf(1.8))) if r % 11 else 0  # every 11th row empty
        if r % 13 == 1:
            cols = rng.choice(n // 2, size=min(k + 3, n // 2), replace=False)  # low half only
        elif r % 13 == 2:
            cols = n // 2 + rng.choice(n - n // 2, size=min(k + 3, n // 2), replace=False)  # high half only
        elif r % 7 == 3:  # long rows straddling the split: unaligned starts, tails across pieces
            lo = (1, 2, 3, 5, 255, 257, 701)[(r // 7) % 7]
            hi = (257, 258, 259, 513, 515, 600)[(r // 49) % 6]
            cols = np.arange(max(0, n // 2 - lo), min(n, n // 2 + hi))
        else:
            cols = rng.choice(n, size=min(k, n), replace=False)
        ent += [(r, int(c), float(rng.uniform(-1, 1))) for c in cols]
    a = _csr(n, n, ent)
    plan = P.inspect(KernelKind.Spmv, a, 3, 8)
    x = P.uniform_vector(n, 5)
    want = Oracle.run_spmv(plan.export_arrays(), a.view(), x)
    bound = P.BoundPlan(exe, plan, a)
    xd = torch.from_numpy(x).cuda()
    yd = torch.full((n,), float("nan"), dtype=torch.float64, device="cuda")
    for _ in range(2):  # the state buffer is reused across calls
        bound.spmv(xd, yd)
    torch.cuda.synchronize()
    assert bitwise_equal(yd.cpu().numpy(), want)
    yh = np.full(n, np.nan)
    bound.spmv_host(x, yh)  # host-buffer path (H2D x, passes, D2H y)
    torch.cuda.synchronize()
    assert bitwise_equal(yh, want)
    assert bound.launches() >= (2 if force else 1)


@pytest.mark.parametrize("layout", ["first_row_long", "all_rows_long", "long_head_short_tail"])
def test_spmv_column_split_host_slices(monkeypatch, layout):
    """The host-buffer path runs the last column pass in row slices and sends
    each slice's y down as it finishes: rows before the first chunk (long rows
    in the last pass) and a last pass with only long rows must be covered too
    (slice 0 started at the first chunk's row)."""
    import torch

    monkeypatch.setenv("PSC_SPMV_SPLIT_BYTES", "1")
    monkeypatch.setenv("PSC_SPMV_SPLIT_PARTS", "2")
    exe = P.Executor(1)
    rng = np.random.default_rng(7)
    n = 1200
    long_rows = {"first_row_long": {0}, "all_rows_long": set(range(0, n, 150)),
                 "long_head_short_tail": set(range(5))}[layout]
    ent = []
    for r in range(n if layout != "all_rows_long" else 8):
        rr = r if layout != "all_rows_long" else r * 150
        if rr in long_rows:
            cols = np.arange(n // 2, n // 2 + 300)  # > 256 entries in the last (upper) column half
            cols = np.concatenate([np.arange(0, 20), cols])
        else:
            cols = rng.choice(n, size=int(rng.integers(1, 6)), replace=False)
        ent += [(rr, int(c), float(rng.uniform(-1, 1))) for c in cols]
    a = _csr(n, n, ent)
    plan = P.inspect(KernelKind.Spmv, a, 3, 8)
    x = P.uniform_vector(n, 9)
    want = Oracle.run_spmv(plan.export_arrays(), a.view(), x)
    bound = P.BoundPlan(exe, plan, a)
    for host in (np.full(n, np.nan), torch.full((n,), float("nan"), dtype=torch.float64).pin_memory().numpy()):
        bound.spmv_host(x, host)
        torch.cuda.synchronize()
        assert bitwise_equal(host, want), layout


def test_spmv_side_stream_concurrent_threads(monkeypatch):
    """Plans that fork work onto the side stream (row groups beside chunks,
    long rows beside chunks, column-split passes) driven from five host
    threads at once, each on its own CUDA stream with its own bound plan; x
    changes on the caller's stream before every call, so a side-stream launch
    that ran ahead of its fork would read a stale x. Bitwise per call."""
    import threading

    import torch

    exe = P.Executor(1)
    a_groups = _block_rows_matrix()
    rng = np.random.default_rng(41)
    n = 2000
    ent = []
    for r in range(n):
        k = 300 if r % 97 == 0 else 6  # long rows (> 256 entries) among chunk rows
        ent += [(r, int(c), float(rng.uniform(-1, 1))) for c in rng.choice(n, size=k, replace=False)]
    a_long = _csr(n, n, ent)
    jobs = []
    for a, split in ((a_groups, "-1"), (a_long, "-1"), (a_long, "1"), (a_groups, "-1"), (a_long, "1")):
        monkeypatch.setenv("PSC_SPMV_SPLIT_BYTES", split)  # read at bind: "1" forces the split passes
        plan = P.inspect(KernelKind.Spmv, a, 3, 8)
        xs = [P.uniform_vector(a.n_cols, 100 + i) for i in range(4)]
        want = [Oracle.run_spmv(plan.export_arrays(), a.view(), x) for x in xs]
        jobs.append((P.BoundPlan(exe, plan, a), xs, want))
    iters = 40
    monkeypatch.setenv("PSC_SPMV_SPLIT_BYTES", "-1")
    results = [None] * len(jobs)

    def run(j):
        bound, xs, _ = jobs[j]
        s = torch.cuda.Stream()
        with torch.cuda.stream(s):
            xsd = [torch.from_numpy(x).cuda() for x in xs]
            xd = torch.empty_like(xsd[0])
            yd = torch.empty(len(jobs[j][2][0]), dtype=torch.float64, device="cuda")
            out = torch.empty((iters, yd.numel()), dtype=torch.float64, device="cuda")
            for i in range(iters):
                xd.copy_(xsd[i % len(xs)])
                bound.spmv(xd, yd, stream=s)
                out[i].copy_(yd)
        s.synchronize()
        results[j] = out.cpu().numpy()

    threads = [threading.Thread(target=run, args=(j,)) for j in range(len(jobs))]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    for j, (_, xs, want) in enumerate(jobs):
        for i in range(iters):
            assert bitwise_equal(results[j][i], want[i % len(xs)]), (j, i)


@pytest.mark.parametrize("n,band", [(5, 2), (1000, 3), (100003, 40), (20000, None)])
def test_spmv_host_row_slices(n, band):
    """Host-buffer SpMV (`psc_bound_spmv_host`) of thread-per-row plans:
    banded rows, a 5-row matrix, random columns, empty rows. Bitwise against
    the oracle, twice in a row (the second call reuses the scratch buffers)."""
    import torch

    rng = np.random.default_rng(n)
    ent = []
    for r in range(n):
        if band is None:
            cols = rng.choice(n, size=min(n, 7), replace=False)
        else:
            cols = [c for c in range(r - band, r + band + 1, max(1, band // 3)) if 0 <= c < n]
        if r % 17 == 5:
            cols = []  # empty rows
        ent += [(r, int(c), float(rng.uniform(-1, 1))) for c in cols]
    a = _csr(n, n, ent)
    exe = P.Executor(1)
    plan = P.inspect(KernelKind.Spmv, a, 3, 8)
    bound = P.BoundPlan(exe, plan, a)
    for seed in (1, 2):
        x = P.uniform_vector(n, seed)
        want = Oracle.run_spmv(plan.export_arrays(), a.view(), x)
        xh = torch.from_numpy(x).pin_memory().numpy()
        yh = torch.full((n,), float("nan"), dtype=torch.float64).pin_memory().numpy()
        bound.spmv_host(xh, yh)
        torch.cuda.synchronize()
        assert bitwise_equal(yh, want), seed


def test_bind_refuses_a_plan_from_another_matrix(exe, tmp_path):
    """A mined plan's tables are its matrix's columns; binding it to a matrix of
    the same shape but another structure is refused -- also after a save /
    load round trip (the file records the structure hash)."""
    a = P.generate_config(1, 0.0004)  # 20 x 20 grid
    b = P.generate_config(1, 0.0004)
    b.col_indices = b.col_indices.copy()
    r = 7
    k0, k1 = int(b.row_offsets[r]), int(b.row_offsets[r + 1])
    b.col_indices[k0] = b.col_indices[k0] - 1 if b.col_indices[k0] > 0 else 1  # still sorted, same nnz
    assert np.all(np.diff(b.col_indices[k0:k1]) > 0)
    plan = P.inspect(KernelKind.Spmv, a, 3, 8)
    P.BoundPlan(exe, plan, a).close()
    with pytest.raises(P.LogicError):
        P.BoundPlan(exe, plan, b)
    path = tmp_path / "a.plan"
    plan.save(path)
    loaded = P.CodeletPlan.load(path, a)
    P.BoundPlan(exe, loaded, a).close()
    with pytest.raises(P.LogicError):
        P.BoundPlan(exe, loaded, b)


def test_run_cache_sees_in_place_structure_edits(exe):
    """run_spmv caches the binding per (plan, arrays); an in-place edit of the
    structure (anywhere -- the check hashes all of it) must rebind, and the
    result must follow the edited matrix (the reference re-reads it)."""
    a = P.generate_config(1, 0.0004)
    x = P.uniform_vector(a.n_cols, 3)
    plan = P.inspect(KernelKind.Spmv, a, 3, 8)
    y = np.empty(a.n_rows)
    P.run_spmv(plan, a, x, y, exe)
    assert bitwise_equal(y, Oracle.run_spmv(plan.export_arrays(), a.view(), x))
    # a structure edit the plan no longer matches: the rebind must refuse it
    k = int(a.row_offsets[250])
    a.col_indices[k] = a.col_indices[k] + 1 if a.col_indices[k] + 1 < a.col_indices[k + 1] else a.col_indices[k]
    if not np.all(np.diff(a.col_indices[a.row_offsets[250]:a.row_offsets[251]]) > 0):
        pytest.skip("edit would unsort the row")
    with pytest.raises((P.LogicError, P.InvalidArgument)):
        P.run_spmv(plan, a, x, y, exe)


@pytest.mark.parametrize("kernel,config,mode", [(0, 5, 1), (1, 2, 0)])
def test_host_buffer_calls_from_threads(kernel, config, mode):
    """psc_bound_*_host calls on one bound from four host threads, each on its
    own stream: the calls share the bound's scratch buffers and are
    serialised, so every thread gets the right result."""
    import threading

    import torch

    exe = P.Executor(1)
    a = P.generate_config(config, 0.002 if config == 5 else 0.05)
    kk = P.KernelKind.Spmv if kernel == 0 else P.KernelKind.Sptrsv
    import os

    if kernel == 0:
        os.environ["PSC_FAST_SPLIT_BYTES"] = "100000"  # several column passes: copy stream + events
    try:
        plan = P.inspect(kk, a, 3, 8)
        bound = P.BoundPlan(exe, plan, a, mode=mode)
    finally:
        os.environ.pop("PSC_FAST_SPLIT_BYTES", None)
    vecs = [P.uniform_vector(a.n_cols, 40 + i) for i in range(4)]
    want = []
    for v in vecs:
        out = np.empty(a.n_rows)
        (bound.spmv_host if kernel == 0 else bound.sptrsv_host)(v, out)
        torch.cuda.synchronize()
        want.append(out)
    errors = []

    def worker(i):
        try:
            s = torch.cuda.Stream()
            for _ in range(5):
                out = np.full(a.n_rows, np.nan)
                (bound.spmv_host if kernel == 0 else bound.sptrsv_host)(vecs[i], out, stream=s)
                s.synchronize()
                if not np.array_equal(out.view(np.int64), want[i].view(np.int64)):
                    errors.append(i)
        except Exception as e:  # noqa: BLE001
            errors.append(repr(e))

    ts = [threading.Thread(target=worker, args=(i,)) for i in range(4)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert not errors, errors
    exe.close()
