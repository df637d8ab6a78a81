"""GPU parity: the sm_100a executor against the C oracle (oracle/psc_oracle.c,
itself pinned bitwise to the reference executor in test_oracle.py).

Bar: bitwise equality with the reference executor's arithmetic (parity mode)
on every plan, exact equality with the naive baseline on integer data
(acceptance_main.cpp:156-157), and the reference's 1e-12 elementwise bound on
the random suite."""
import numpy as np
import pytest

import paper_2111_12243_b200 as P
from oracle.oracle import Oracle
from paper_2111_12243_b200 import KernelKind
from tests.helpers import bitwise_equal, max_rel_err, normwise_err, suite_cases, suite_input, pattern

pytestmark = pytest.mark.gpu


def run_gpu(exe, plan, kernel, a, vec):
    if kernel == KernelKind.Spmv:
        y = np.full(a.n_rows, np.nan)
        P.run_spmv(plan, a, vec, y, exe)
        return y
    x = np.full(a.n_rows, np.nan)
    acc = np.full(a.n_rows, np.nan)
    P.run_sptrsv(plan, P.TriangularMatrix.adopt(a), vec, x, acc, exe)
    return x


def run_oracle(plan, kernel, a, vec):
    if kernel == KernelKind.Spmv:
        return Oracle.run_spmv(plan.export_arrays(), a.view(), vec)
    return Oracle.run_sptrsv(plan.export_arrays(), a.view(), vec)[0]


def baseline(kernel, a, vec):
    if kernel == KernelKind.Spmv:
        return Oracle.spmv_baseline(a.view(), vec)
    return Oracle.sptrsv_baseline(a.view(), vec)


def test_acceptance_suite_bitwise(exe):
    """acceptance_main.cpp:127-174: 42 cases x t in {1,2,3,8} x groups in {1,4} = 336 plans."""
    n_plans = mismatches = 0
    for name, kernel, a, ints in suite_cases():
        vec = suite_input(kernel, a, ints)
        want = baseline(kernel, a, vec)
        for t in (1, 2, 3, 8):
            for groups in (1, 4):
                plan = P.inspect(kernel, a, t, groups)
                got = run_gpu(exe, plan, kernel, a, vec)
                ref = run_oracle(plan, kernel, a, vec)
                assert bitwise_equal(got, ref), f"{name} t={t} groups={groups}: not bitwise equal to the executor"
                ok = bitwise_equal(got, want) if ints else max_rel_err(got, want) <= 1e-12
                mismatches += 0 if ok else 1
                n_plans += 1
    assert n_plans == 336 and mismatches == 0


@pytest.mark.parametrize("config,scale,kernel", [
    (1, 1.0, KernelKind.Spmv),
    (2, 1.0, KernelKind.Sptrsv),
    (3, 0.05, KernelKind.Spmv),
    (4, 0.1, KernelKind.Sptrsv),
    (5, 0.02, KernelKind.Spmv),
])
def test_configs_bitwise(exe, config, scale, kernel):
    a = P.generate_config(config, scale)
    plan = P.inspect(kernel, a, 3, 8)
    vec = P.uniform_vector(a.n_cols, 10 + config)
    got = run_gpu(exe, plan, kernel, a, vec)
    assert bitwise_equal(got, run_oracle(plan, kernel, a, vec))
    tol = 1e-12 if kernel == KernelKind.Spmv else 1e-10
    assert normwise_err(got, baseline(kernel, a, vec)) <= tol


@pytest.mark.parametrize("config,kernel", [(3, KernelKind.Spmv), (4, KernelKind.Sptrsv), (5, KernelKind.Spmv)])
def test_configs_full_size_bitwise(exe, config, kernel):
    """acceptance_main.cpp:127-174 criterion 1 at BASELINE.json's full sizes,
    where the production paths engage: config 3's row groups and quad chunks,
    config 4's streaming long-row solve, config 5's column-split passes (x =
    160 MB) and long rows -- through the host-span API (run_spmv /
    run_sptrsv) and, for the SpMV configs, the bound device and host-buffer
    paths."""
    import torch

    a = P.generate_config(config, 1.0)
    plan = P.inspect(kernel, a, 3, 8)
    vec = P.uniform_vector(a.n_cols, 10 + config)
    want = run_oracle(plan, kernel, a, vec)
    got = run_gpu(exe, plan, kernel, a, vec)
    assert bitwise_equal(got, want)
    tol = 1e-12 if kernel == KernelKind.Spmv else 1e-10
    assert normwise_err(got, baseline(kernel, a, vec)) <= tol
    if kernel == KernelKind.Spmv:
        bound = P.BoundPlan(exe, plan, a)
        if config == 5:
            assert bound.info()["passes_or_block_rows"] >= 2  # column-split passes engaged
        xd = torch.from_numpy(vec).cuda()
        yd = torch.full((a.n_rows,), float("nan"), dtype=torch.float64, device="cuda")
        bound.spmv(xd, yd)
        torch.cuda.synchronize()
        assert bitwise_equal(yd.cpu().numpy(), want)
        xp = torch.from_numpy(vec).pin_memory()
        yp = torch.full((a.n_rows,), float("nan"), dtype=torch.float64).pin_memory()
        bound.spmv_host(xp.numpy(), yp.numpy())
        torch.cuda.synchronize()
        assert bitwise_equal(yp.numpy(), want)
        bound.close()


def test_bound_device_path_matches_host_path(exe):
    import torch

    a = P.generate_config(2, 0.02)
    plan = P.inspect(KernelKind.Sptrsv, a, 3, 8)
    b = P.uniform_vector(a.n_rows, 3)
    host = run_gpu(exe, plan, KernelKind.Sptrsv, a, b)
    bound = P.BoundPlan(exe, plan, a)
    bd = torch.from_numpy(b).cuda()
    xd = torch.empty_like(bd)
    accd = torch.empty_like(bd)
    for _ in range(3):  # repeated solves re-arm correctly
        bound.sptrsv(bd, xd, accd)
    torch.cuda.synchronize()
    assert bitwise_equal(xd.cpu().numpy(), host)
    xh = np.empty_like(b)
    bound.sptrsv_host(b, xh)
    torch.cuda.synchronize()
    assert bitwise_equal(xh, host)
    # pinned (mapped) host buffers: the solve writes x to host memory directly
    bp = torch.from_numpy(b).pin_memory()
    xp = torch.full((a.n_rows,), float("nan"), dtype=torch.float64).pin_memory()
    accp = torch.full((a.n_rows,), float("nan"), dtype=torch.float64).pin_memory()
    for _ in range(2):
        bound.sptrsv_host(bp.numpy(), xp.numpy(), accp.numpy())
        torch.cuda.synchronize()
        assert bitwise_equal(xp.numpy(), host)
        assert bitwise_equal(accp.numpy(), accd.cpu().numpy())


# ---- exec_*_codelet known answers (test_executor.cpp:37-114) ----

def _ctx(ax, x, acc, rhs=None):
    return P.ExecutionContext(np.array(ax, float), np.array(x, float), acc, rhs)


def test_blas_codelet_known_answers():
    c = P.Codelet(P.CodeletKind.Blas, 3, 3, P.AccessDesc.strided(0, 1, 0), P.AccessDesc.strided(0, 3, 1),
                  P.AccessDesc.strided(0, 0, 1))
    acc = np.zeros(3)
    P.exec_blas_codelet(c, _ctx(range(1, 10), [1, 1, 1], acc))
    assert acc.tolist() == [6, 15, 24]
    c.vec = P.AccessDesc.strided(0, 0, 2)  # non-unit inner stride: sequential branch
    acc = np.zeros(3)
    P.exec_blas_codelet(c, _ctx(range(1, 10), [1, 0, 1, 0, 1, 0], acc))
    assert acc.tolist() == [6, 15, 24]
    one = P.Codelet(P.CodeletKind.Blas, 1, 1, P.AccessDesc.strided(2, 0, 0), P.AccessDesc.strided(1, 0, 1),
                    P.AccessDesc.strided(3, 0, 1))
    acc = np.ones(3)
    P.exec_blas_codelet(one, _ctx([0, 5, 0], [0, 0, 0, 4], acc))
    assert acc.tolist() == [1, 1, 21]


def test_psc_codelet_known_answers():
    c = P.Codelet(P.CodeletKind.PscI, 3, 3, P.AccessDesc.strided(0, 1, 0), P.AccessDesc.strided(0, 3, 1),
                  P.AccessDesc.inner_table([0, 2, 5]))
    acc = np.zeros(3)
    P.exec_psci_codelet(c, _ctx(range(1, 10), [10, 0, 20, 0, 0, 30], acc))
    assert acc.tolist() == [140, 320, 500]
    c2 = P.Codelet(P.CodeletKind.PscII, 1, 2, P.AccessDesc.outer_table([0]), P.AccessDesc.strided(0, 0, 1),
                   P.AccessDesc.inner_table([1, 3]))
    acc = np.zeros(1)
    P.exec_pscii_codelet(c2, _ctx([2, 5], [0, 1, 0, 1], acc))
    assert acc.tolist() == [7]
    f = P.Codelet(P.CodeletKind.PscII, 2, 1, P.AccessDesc.outer_table([0, 1]), P.AccessDesc.strided(0, 1, 1),
                  P.AccessDesc.point_table([1, 3]))
    acc = np.zeros(2)
    P.exec_pscii_codelet(f, _ctx([2, 5], [0, 1, 0, 1], acc))
    assert acc.tolist() == [2, 5]


def test_codelet_shape_errors():
    """test_executor.cpp:116-138."""
    c = P.Codelet(P.CodeletKind.Blas, 1, 1, P.AccessDesc.strided(0, 0, 0), P.AccessDesc.strided(0, 0, 1),
                  P.AccessDesc.inner_table([0]))
    ctx = _ctx([1], [1], np.zeros(1))
    with pytest.raises(P.InvalidArgument):
        P.exec_blas_codelet(c, ctx)
    c.vec = P.AccessDesc.strided(0, 0, 1)
    with pytest.raises(P.InvalidArgument):
        P.exec_psci_codelet(c, ctx)
    with pytest.raises(P.InvalidArgument):
        P.exec_pscii_codelet(c, ctx)
    c.out, c.mat, c.vec = P.AccessDesc.outer_table([0]), P.AccessDesc.inner_table([0]), P.AccessDesc.inner_table([0])
    with pytest.raises(P.InvalidArgument):
        P.exec_pscii_codelet(c, ctx)


@pytest.mark.parametrize("world", [2, 4, 8])
def test_partition_shards_bitwise(exe, world):
    """Row shards bound by partition (multi-GPU path) equal the full plan's rows."""
    import torch

    from paper_2111_12243_b200.dist import shard_partitions

    a = P.generate_config(5, 0.01)
    plan = P.inspect(KernelKind.Spmv, a, 3, 8)
    x = P.uniform_vector(a.n_cols, 15)
    want = Oracle.run_spmv(plan.export_arrays(), a.view(), x)
    xd = torch.from_numpy(x).cuda()
    n_parts = plan.counts().n_partitions
    for r in range(world):
        p0, p1 = shard_partitions(n_parts, world, r)
        if p1 == p0:
            continue
        bound = P.BoundPlan(exe, plan, a, partitions=(p0, p1))
        y = torch.empty(bound.row_end - bound.row_begin, dtype=torch.float64, device="cuda")
        bound.spmv(xd, y)
        torch.cuda.synchronize()
        assert bitwise_equal(y.cpu().numpy(), want[bound.row_begin:bound.row_end])


@pytest.mark.parametrize("config,scale", [(1, 0.25), (5, 0.01), (1, 0.002)])
@pytest.mark.parametrize("world", [2, 4, 8])
def test_fused_peer_exchange_bitwise(exe, config, scale, world):
    """The fused exchange + multiply (psc_bound_spmv_peers): every "rank" has
    its own x window on this GPU holding only its own entries; each shard's
    launch pulls the columns it reads from the other windows and multiplies.
    Stitched shards equal the full plan bitwise, twice in a row (the pull
    counters advance per launch), and each window ends up holding exactly x
    on the runs its shard reads. No launch waits on another launch."""
    import torch

    from paper_2111_12243_b200.dist import shard_partitions

    a = P.generate_config(config, scale)
    plan = P.inspect(KernelKind.Spmv, a, 3, 8)
    x = P.uniform_vector(a.n_cols, 21)
    want = Oracle.run_spmv(plan.export_arrays(), a.view(), x)
    n_parts = plan.counts().n_partitions
    bounds, ranges = [], []
    for r in range(world):
        p0, p1 = shard_partitions(n_parts, world, r)
        assert p1 > p0
        bounds.append(P.BoundPlan(exe, plan, a, partitions=(p0, p1)))
        ranges.append((bounds[-1].row_begin, bounds[-1].row_end))
    xt = torch.from_numpy(x).cuda()
    windows = []
    for (b, e) in ranges:
        w = torch.full((a.n_cols,), float("nan"), dtype=torch.float64, device="cuda")
        w[b:e] = xt[b:e]
        windows.append(w)
    peers = [(windows[q].data_ptr(), b, e) for q, (b, e) in enumerate(ranges)]
    for _ in range(2):
        ys = []
        for q, bound in enumerate(bounds):
            y = torch.full((ranges[q][1] - ranges[q][0],), float("nan"), dtype=torch.float64, device="cuda")
            bound.spmv_peers(peers, windows[q], y)
            ys.append(y)
        torch.cuda.synchronize()
        got = torch.cat(ys).cpu().numpy()
        assert bitwise_equal(got, want)
    for q, bound in enumerate(bounds):
        w = windows[q].cpu().numpy()
        for c0, c1 in bound.x_runs():
            assert bitwise_equal(w[c0:c1], x[c0:c1])


def test_general_path_hand_built_plan(exe):
    """A hand-built plan that is not canonical (shared out table, strided gather)
    runs through the exact interpreter and matches the oracle bitwise."""
    a = pattern("dense_block(4)")
    # rows 0 and 1 of the matrix accumulate into outputs 1 and 0 (crossed): not canonical
    c1 = P.Codelet(P.CodeletKind.Blas, 2, 4, P.AccessDesc.strided(1, -1, 0), P.AccessDesc.strided(0, 4, 1),
                   P.AccessDesc.strided(0, 0, 1))
    c2 = P.Codelet(P.CodeletKind.PscII, 2, 4, P.AccessDesc.outer_table([2, 3]), P.AccessDesc.strided(8, 4, 1),
                   P.AccessDesc.point_table([0, 1, 2, 3, 0, 1, 2, 3]))
    g = P.RegionGroup(P.RowWindow(0, 4), P.MineStrategy.BlasFirst, 0, [c2, c1], [])
    plan = P.CodeletPlan.from_partitions(KernelKind.Spmv, 4, 4, 16, 4, 1, [P.PartitionPlan([g])])
    x = np.array([1.0, 2.0, 3.0, 4.0])
    y = np.zeros(4)
    P.run_spmv(plan, a, x, y, exe)
    assert bitwise_equal(y, Oracle.run_spmv(plan.export_arrays(), a.view(), x))
    ctx = P.ExecutionContext(a.values.copy(), x.copy(), np.ones(4))
    exe.run(plan, ctx, a)  # execute_plan: accumulates onto accum
    want = np.ones(4) + Oracle.run_spmv(plan.export_arrays(), a.view(), x)
    assert np.allclose(ctx.accum, want)


def test_division_matches_ieee():
    """The solve kernels divide with a precomputed reciprocal and the final
    correction of the IEEE division (kernels.cu div_with_rcp); it must agree
    bitwise with __ddiv_rn everywhere, including the fallback range."""
    from paper_2111_12243_b200 import _capi
    import ctypes as C
    for seed, span in ((1, 60), (2, 500), (3, 1000)):
        bad = C.c_int64(-1)
        st = _capi.lib().psc_selftest_division(seed, 20_000_000, span, C.byref(bad))
        assert st == 0, _capi.lib().psc_last_error()
        assert bad.value == 0, (span, bad.value)


@pytest.mark.parametrize("lean", ["2", "4", "4-generic-triangle"])
@pytest.mark.parametrize("block_rows", ["1024", "0"])
def test_sptrsv_round_kernels_bitwise(monkeypatch, lean, block_rows):
    """Both solve kernels (records where they apply, PSC_TRSV_LEAN=2; the
    streaming / unit queue, 4 -- with its dense triangle phase and with the
    generic one only, PSC_TRSV_DENSE=0), with default and small blocks (many
    operands from earlier blocks), equal the oracle."""
    if lean.endswith("generic-triangle"):
        monkeypatch.setenv("PSC_TRSV_DENSE", "0")
        lean = "4"
    monkeypatch.setenv("PSC_TRSV_LEAN", lean)
    if block_rows != "0":
        monkeypatch.setenv("PSC_SPTRSV_BLOCK_ROWS", block_rows)
    for config, scale in ((2, 0.03), (4, 0.02), (3, 0.01), (1, 0.002)):
        a = P.generate_config(config, scale)
        if config in (1, 3):  # SpMV matrices: solve with their lower triangle
            a = P.lower_triangular(a).csr()
        plan = P.inspect(KernelKind.Sptrsv, a, 3, 8)
        b = P.uniform_vector(a.n_rows, 5)
        exe = P.Executor(1)
        got = run_gpu(exe, plan, KernelKind.Sptrsv, a, b)
        want = run_oracle(plan, KernelKind.Sptrsv, a, b)
        assert bitwise_equal(got, want), (config, lean, block_rows)


def test_sptrsv_value_update_repacks(exe):
    """run_sptrsv re-uploads values on every call (the reference reads them
    live); the per-row records must follow."""
    a = P.generate_config(2, 0.03)
    plan = P.inspect(KernelKind.Sptrsv, a, 3, 8)
    b = P.uniform_vector(a.n_rows, 9)
    first = run_gpu(exe, plan, KernelKind.Sptrsv, a, b)
    assert bitwise_equal(first, run_oracle(plan, KernelKind.Sptrsv, a, b))
    a.values[:] = a.values * 0.5 + 0.25
    second = run_gpu(exe, plan, KernelKind.Sptrsv, a, b)
    assert bitwise_equal(second, run_oracle(plan, KernelKind.Sptrsv, a, b))
    assert not bitwise_equal(first, second)


def _ipc_worker(rank, world, port, q, mode=0):
    import os

    import torch
    import torch.distributed as dist

    from paper_2111_12243_b200.dist import PeerExchange, shard_partitions, shard_row_ranges

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    if mode == 1:
        os.environ["PSC_FAST_SPLIT_BYTES"] = "400000"  # several column passes
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        a = P.generate_config(5, 0.005)
        plan = P.inspect(KernelKind.Spmv, a, 3, 8)
        p0, p1 = shard_partitions(plan.counts().n_partitions, world, rank)
        bound = P.BoundPlan(P.Executor(1, 0), plan, a, mode=mode, partitions=(p0, p1))
        ranges = shard_row_ranges(plan, world)
        ex = PeerExchange(bound, ranges, rank, a.n_cols, device=torch.device("cpu"))
        x = torch.from_numpy(P.uniform_vector(a.n_cols, 31)).cuda()
        b, e = ranges[rank]
        outs = []
        for _ in range(2):
            y = torch.full((e - b,), float("nan"), dtype=torch.float64, device="cuda")
            ex.multiply(x[b:e].contiguous(), y)
            torch.cuda.synchronize()
            outs.append(y.cpu().numpy())
        y = torch.empty(e - b, dtype=torch.float64, device="cuda")
        bound.spmv(x, y)  # the shard's multiply on the whole x, for comparison
        torch.cuda.synchronize()
        outs.append(y.cpu().numpy())
        dist.barrier()
        ex.close()
        q.put((rank, outs))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("mode", [0, 1])
def test_peer_exchange_real_ipc_two_processes(mode):
    """Two processes on this GPU exchange real CUDA IPC windows (gloo for the
    control plane) and multiply their shards through the fused launch (parity
    mode) or copy-engine pulls per column pass (fast mode); parity: the
    stitched result equals the oracle bitwise; fast: every shard equals its
    multiply on the whole x bitwise, and the stitched result is within 1e-12
    normwise of the reference baseline. The processes' kernels never wait on
    each other (each waits only for its own pulls)."""
    import socket

    import torch.multiprocessing as mp

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_ipc_worker, args=(r, world, port, q, mode)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in range(world))
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    a = P.generate_config(5, 0.005)
    plan = P.inspect(KernelKind.Spmv, a, 3, 8)
    x = P.uniform_vector(a.n_cols, 31)
    if mode == 0:
        want = Oracle.run_spmv(plan.export_arrays(), a.view(), x)
        for it in range(2):
            got = np.concatenate([res[r][it] for r in range(world)])
            assert bitwise_equal(got, want)
    else:
        from tests.helpers import normwise_err

        for r in range(world):
            assert bitwise_equal(res[r][0], res[r][2]) and bitwise_equal(res[r][1], res[r][2]), r
        got = np.concatenate([res[r][0] for r in range(world)])
        assert normwise_err(got, Oracle.spmv_baseline(a.view(), x)) <= 1e-12


# ---- GPU inspector (psc_inspect_device): the same plans as the host inspector ----

def test_device_inspector_acceptance_suite():
    """Every plan of the acceptance suite (42 cases x t x groups) mined on the
    GPU has the host inspector's digest (which is pinned to the reference's
    own inspector in test_oracle.py)."""
    n = 0
    for name, kernel, a, _ in suite_cases():
        for t in (1, 2, 3, 8):
            for groups in (1, 4):
                want = P.inspect(kernel, a, t, groups).hash()
                got = P.inspect_device(kernel, a, t, groups).hash()
                assert got == want, f"{name} t={t} groups={groups}"
                n += 1
    assert n == 336


@pytest.mark.parametrize("config,scale,kernel", [
    (1, 1.0, KernelKind.Spmv),
    (2, 1.0, KernelKind.Sptrsv),
    (3, 0.2, KernelKind.Spmv),
    (4, 0.5, KernelKind.Sptrsv),
    (5, 0.05, KernelKind.Spmv),
])
def test_device_inspector_configs(config, scale, kernel):
    a = P.generate_config(config, scale)
    host = P.inspect(kernel, a, 3, 8)
    dev = P.inspect_device(kernel, a, 3, 8)
    assert dev.hash() == host.hash()
    assert dev.counts().n_codelets == host.counts().n_codelets
    assert dev.totals() == host.totals()


@pytest.mark.parametrize("kernel", [KernelKind.Spmv, KernelKind.Sptrsv])
def test_values_version_skips_reupload(kernel):
    """psc_executor_set_values_version: untagged calls read the values live (as
    the reference does); a call tagged with the version already on the device
    keeps those values; a new tag uploads again."""
    exe = P.Executor(1)
    a = P.generate_config(2 if kernel == KernelKind.Sptrsv else 1, 0.02)
    plan = P.inspect(kernel, a, 3, 8)
    v = P.uniform_vector(a.n_rows, 3)
    first = run_gpu(exe, plan, kernel, a, v)
    assert bitwise_equal(first, run_oracle(plan, kernel, a, v))
    a.values[:] *= 0.5  # in place, same arrays
    live = run_gpu(exe, plan, kernel, a, v)
    assert bitwise_equal(live, run_oracle(plan, kernel, a, v))  # untagged: re-uploaded
    exe.set_values_version(7)
    tagged = run_gpu(exe, plan, kernel, a, v)  # first call with tag 7 uploads
    assert bitwise_equal(tagged, live)
    a.values[:] *= 2.0
    kept = run_gpu(exe, plan, kernel, a, v)  # same tag: the device keeps the halved values
    assert bitwise_equal(kept, live)
    exe.set_values_version(8)
    again = run_gpu(exe, plan, kernel, a, v)
    assert bitwise_equal(again, first)
    exe.close()


@pytest.mark.parametrize("split_bytes", ["-1", "500000"])
@pytest.mark.parametrize("world", [2, 4, 8])
def test_fused_peer_exchange_fast_mode(monkeypatch, exe, split_bytes, world):
    """Fast-mode shards (config 5's entry streams, one or several column
    passes): psc_bound_spmv_peers pulls each pass's remote runs with the copy
    engines and runs the pass after its own range landed. Every shard equals
    its own multiply on the fully gathered x bitwise, twice in a row, and the
    stitched result is within 1e-12 normwise of the reference baseline."""
    import torch

    from paper_2111_12243_b200.dist import shard_partitions
    from tests.helpers import normwise_err

    monkeypatch.setenv("PSC_FAST_SPLIT_BYTES", split_bytes)
    a = P.generate_config(5, 0.01)
    plan = P.inspect(KernelKind.Spmv, a, 3, 8)
    x = P.uniform_vector(a.n_cols, 23)
    xt = torch.from_numpy(x).cuda()
    n_parts = plan.counts().n_partitions
    bounds, ranges = [], []
    for r in range(world):
        p0, p1 = shard_partitions(n_parts, world, r)
        bounds.append(P.BoundPlan(exe, plan, a, mode=1, partitions=(p0, p1)))
        ranges.append((bounds[-1].row_begin, bounds[-1].row_end))
        assert bounds[-1].info()["path"] == 2
    windows = []
    for (b, e) in ranges:
        w = torch.full((a.n_cols,), float("nan"), dtype=torch.float64, device="cuda")
        w[b:e] = xt[b:e]
        windows.append(w)
    peers = [(windows[q].data_ptr(), b, e) for q, (b, e) in enumerate(ranges)]
    ref = []
    for q, bound in enumerate(bounds):
        y = torch.empty(ranges[q][1] - ranges[q][0], dtype=torch.float64, device="cuda")
        bound.spmv(xt, y)
        ref.append(y)
    for _ in range(2):
        ys = []
        for q, bound in enumerate(bounds):
            y = torch.full((ranges[q][1] - ranges[q][0],), float("nan"), dtype=torch.float64, device="cuda")
            bound.spmv_peers(peers, windows[q], y)
            ys.append(y)
        torch.cuda.synchronize()
        for q in range(world):
            assert bitwise_equal(ys[q].cpu().numpy(), ref[q].cpu().numpy()), q
    got = torch.cat(ys).cpu().numpy()
    assert normwise_err(got, Oracle.spmv_baseline(a.view(), x)) <= 1e-12
