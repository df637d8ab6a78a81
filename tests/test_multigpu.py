"""Multi-GPU SpMV host path on CPU: world_size-2 gloo processes shard the plan
by partitions, all-gather x from the owners' slices, and the
stitched row shards equal the single-process result. The per-shard GPU
kernel is covered in tests/test_gpu_parity.py::test_partition_shards_*."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

import paper_2111_12243_b200 as P
from paper_2111_12243_b200.dist import XExchange, shard_partitions, shard_row_ranges


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    import torch
    import torch.distributed as dist

    from oracle.oracle import Oracle

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        a = P.generate_config(5, 0.0005)
        plan = P.inspect(P.KernelKind.Spmv, a, 3, 8)
        ranges = shard_row_ranges(plan, world)
        b, e = ranges[rank]
        x = P.uniform_vector(a.n_cols, 15)
        ex = XExchange(ranges, a.n_cols, device="cpu")
        full = ex.exchange(torch.from_numpy(x[b:e].copy()))
        ok_x = bool(np.array_equal(full.numpy(), x))
        # local rows of y = A x (oracle restricted to this shard's rows)
        y_local = Oracle.run_spmv(plan.export_arrays(), a.view(), full.numpy())[b:e]
        parts = [torch.zeros(max(r[1] - r[0] for r in ranges), dtype=torch.float64) for _ in range(world)]
        mine = torch.zeros_like(parts[0])
        mine[: e - b] = torch.from_numpy(y_local)
        dist.all_gather(parts, mine)
        if rank == 0:
            y = np.concatenate([parts[r][: ranges[r][1] - ranges[r][0]].numpy() for r in range(world)])
            want = Oracle.run_spmv(plan.export_arrays(), a.view(), x)
            q.put((ok_x, bool(np.array_equal(y.view(np.int64), want.view(np.int64))), ranges))
    finally:
        dist.destroy_process_group()


def test_shard_partitions_tile_the_plan():
    for n_parts in (1, 3, 8):
        for world in (1, 2, 4, 8):
            spans = [shard_partitions(n_parts, world, r) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == n_parts
            assert all(spans[i][1] == spans[i + 1][0] for i in range(world - 1))
    a = P.generate_config(1, 0.01)
    plan = P.inspect(P.KernelKind.Spmv, a, 3, 8)
    for world in (1, 2, 4, 8):
        ranges = shard_row_ranges(plan, world)
        assert ranges[0][0] == 0 and ranges[-1][1] == a.n_rows
        assert all(ranges[i][1] == ranges[i + 1][0] for i in range(world - 1))


@pytest.mark.timeout(300)
def test_two_process_gloo_sharded_spmv():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    ok_x, ok_y, ranges = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
    assert ok_x, "all-gathered x differs from the original"
    assert ok_y, "stitched shard results differ from the single-process executor"
    assert len(ranges) == 2


class _FakeIpc:
    """Stands in for CUDA IPC: handles name the owner rank's window."""

    calls = []

    @staticmethod
    def alloc(nbytes):
        import torch.distributed as dist

        r = dist.get_rank()
        return 1000 + r, f"h{r}".encode().ljust(64, b"\0")

    @staticmethod
    def open(handle):
        return 5000 + int(handle.rstrip(b"\0")[1:])

    @staticmethod
    def close(ptr):
        _FakeIpc.calls.append(("close", ptr))

    @staticmethod
    def free(ptr):
        _FakeIpc.calls.append(("free", ptr))

    @staticmethod
    def copy(dst, src, nbytes, stream):
        _FakeIpc.calls.append(("copy", dst, nbytes))


class _FakeBound:
    def __init__(self):
        self.calls = []

    def spmv_peers(self, peers, window, y, stream=None):
        self.calls.append((list(peers), window))


def _peer_worker(rank, world, port, q):
    import torch
    import torch.distributed as dist

    from paper_2111_12243_b200.dist import PeerExchange

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        ranges = [(0, 7), (7, 10)]
        bound = _FakeBound()
        ex = PeerExchange(bound, ranges, rank, 10, ipc=_FakeIpc, device=torch.device("cpu"))
        x_local = torch.zeros(ranges[rank][1] - ranges[rank][0], dtype=torch.float64)
        ex.multiply(x_local, torch.zeros(1, dtype=torch.float64), stream=0)
        ex.close()
        q.put((rank, ex.peers, bound.calls, _FakeIpc.calls))
    finally:
        dist.destroy_process_group()


def test_peer_exchange_host_protocol():
    """PeerExchange with fake IPC on 2 gloo processes: every rank's peer table
    lists its own window and the opened handles of the others in rank order,
    copies its own slice into its window at the right offset, then launches
    once with that table; closes what it opened and frees its window."""
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_peer_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    ranges = [(0, 7), (7, 10)]
    for rank, peers, calls, ipc_calls in res:
        want = [((1000 + q) if q == rank else (5000 + q), b, e) for q, (b, e) in enumerate(ranges)]
        assert peers == want
        assert calls == [(want, 1000 + rank)]
        b = ranges[rank][0]
        assert ipc_calls[0] == ("copy", 1000 + rank + 8 * b, 8 * (ranges[rank][1] - b))
        other = 1 - rank
        assert ("close", 5000 + other) in ipc_calls and ("free", 1000 + rank) in ipc_calls
