"""Multi-GPU SpMV: one process per GPU, row shards = whole plan partitions.

SURVEY.md §8e: the SpMV plan's partitions are contiguous nnz-balanced row
ranges (scheduler.cpp:67-89) and windows never cross them (miner.cpp:298-300),
so rank r executes partitions [r*P/N, (r+1)*P/N) -- an exact slice of the one
bit-exact plan -- and owns the x entries of its rows. A step gathers the full
x and multiplies. Two exchanges:

* ``PeerExchange`` (the default on GPUs): every rank publishes a full-length
  x window as CUDA IPC memory; one fused launch (psc_bound_spmv_peers) pulls
  exactly the columns the shard reads from the peers' windows over NVLink
  while the work on its own columns proceeds;
* ``XExchange``: NCCL all-gather of padded slices (gloo on CPU), then the
  multiply.

Results are bitwise those of the single-GPU executor because every row is
computed by the same code on the same operands. The solve does not shard
(replicas only).
"""
from __future__ import annotations

from typing import List, Tuple

from .psc import CodeletPlan, partition_rows


def shard_partitions(n_partitions: int, world: int, rank: int) -> Tuple[int, int]:
    """Partitions [p0, p1) owned by `rank` (contiguous, as even as possible)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("shard_partitions: bad rank/world")
    return rank * n_partitions // world, (rank + 1) * n_partitions // world


def shard_row_ranges(plan: CodeletPlan, world: int) -> List[Tuple[int, int]]:
    """Row range of every rank's shard."""
    n_parts = plan.counts().n_partitions
    out = []
    for r in range(world):
        p0, p1 = shard_partitions(n_parts, world, r)
        out.append(partition_rows(plan, p0, p1) if p1 > p0 else (0, 0))
    return out


class XExchange:
    """All-gather of the distributed x: rank r holds x[rows_r]; every rank
    receives the full vector. Slices are padded to the largest one so the
    collective is a single all-gather (NCCL all_gather_into_tensor on GPU)."""

    def __init__(self, ranges: List[Tuple[int, int]], n_cols: int, device, dtype=None):
        import torch

        self.ranges = ranges
        self.sizes = [e - b for b, e in ranges]
        self.pad = max(self.sizes) if self.sizes else 0
        self.world = len(ranges)
        dtype = dtype or torch.float64
        self.local = torch.zeros(max(self.pad, 1), dtype=dtype, device=device)
        self.gathered = torch.empty(max(self.pad, 1) * self.world, dtype=dtype, device=device)
        self.full = torch.empty(n_cols, dtype=dtype, device=device)
        if sum(self.sizes) != n_cols or any(b != (ranges[i - 1][1] if i else 0) for i, (b, _) in enumerate(ranges)):
            raise ValueError("XExchange: row shards must tile x contiguously")

    def exchange(self, x_local, group=None):
        """x_local: this rank's slice (len = its rows). Returns the full x."""
        import torch
        import torch.distributed as dist

        n = x_local.numel()
        self.local[:n].copy_(x_local)
        if self.local.is_cuda:
            dist.all_gather_into_tensor(self.gathered, self.local, group=group)
        else:  # gloo
            parts = list(self.gathered.view(self.world, -1).unbind(0))
            dist.all_gather(parts, self.local, group=group)
        g = self.gathered.view(self.world, -1)
        for r, (b, e) in enumerate(self.ranges):
            if e > b:
                self.full[b:e].copy_(g[r, : e - b])
        return self.full


class CudaIpc:
    """CUDA IPC through the C ABI (psc_ipc_*)."""

    @staticmethod
    def alloc(nbytes: int):
        import ctypes as C

        from . import _capi
        from .psc import _check

        ptr, handle = C.c_void_p(), C.create_string_buffer(64)
        _check(_capi.lib().psc_ipc_alloc(int(nbytes), C.byref(ptr), handle))
        return int(ptr.value), bytes(handle.raw)

    @staticmethod
    def open(handle: bytes) -> int:
        import ctypes as C

        from . import _capi
        from .psc import _check

        ptr = C.c_void_p()
        _check(_capi.lib().psc_ipc_open(C.create_string_buffer(handle, 64), C.byref(ptr)))
        return int(ptr.value)

    @staticmethod
    def close(ptr: int) -> None:
        from . import _capi

        _capi.lib().psc_ipc_close(ptr)

    @staticmethod
    def free(ptr: int) -> None:
        from . import _capi

        _capi.lib().psc_ipc_free(ptr)

    @staticmethod
    def copy(dst: int, src: int, nbytes: int, stream) -> None:
        import ctypes as C

        from . import _capi
        from .psc import _check

        _check(_capi.lib().psc_copy_async(C.c_void_p(dst), C.c_void_p(src), int(nbytes), stream))


class PeerExchange:
    """Fused x exchange over peer memory for a row-sharded SpMV.

    Every rank allocates a full-length x window as IPC memory and all-gathers
    the handles; the peer table lists every rank's window (opened over
    NVLink) and row range in rank order. ``multiply`` then:

    1. waits until every rank's previous multiply is done (a one-element
       all-reduce on the stream -- windows are about to be rewritten);
    2. copies this rank's x entries into its window;
    3. waits until every rank has written its window (second all-reduce);
    4. runs the fused launch, which pulls the shard's remote columns from the
       peers' windows and multiplies.
    """

    def __init__(self, bound, ranges: List[Tuple[int, int]], rank: int, n_cols: int, group=None, ipc=None,
                 device=None):
        import torch
        import torch.distributed as dist

        self.bound, self.ranges, self.rank, self.group = bound, ranges, rank, group
        self.ipc = ipc or CudaIpc
        if sum(e - b for b, e in ranges) != n_cols or any(
                b != (ranges[i - 1][1] if i else 0) for i, (b, _) in enumerate(ranges)):
            raise ValueError("PeerExchange: row shards must tile x contiguously")
        try:
            self.window, handle = self.ipc.alloc(8 * max(n_cols, 1))
        except Exception:  # every rank must reach the all-gather; fail together below
            self.window, handle = 0, None
        handles = [None] * len(ranges)
        dist.all_gather_object(handles, handle, group=group)
        self.opened = {}
        if any(h is None for h in handles):
            self.close()
            raise RuntimeError("PeerExchange: IPC allocation failed on a rank")
        peers = []
        for q, (b, e) in enumerate(ranges):
            if q == rank:
                ptr = self.window
            else:
                ptr = self.ipc.open(handles[q])  # a failure here is reported to the caller (bench: all-reduced)
                self.opened[q] = ptr
            peers.append((ptr, b, e))
        self.peers = peers
        dev = device if device is not None else (torch.device("cuda", torch.cuda.current_device())
                                                 if torch.cuda.is_available() else torch.device("cpu"))
        self.token = torch.zeros(1, dtype=torch.float32, device=dev)

    def _sync(self):
        import torch
        import torch.distributed as dist

        if not self.token.is_cuda and torch.cuda.is_available():
            torch.cuda.current_stream().synchronize()  # a host-side collective (gloo) orders nothing on the GPU
        dist.all_reduce(self.token, group=self.group)

    def multiply(self, x_local, y, stream=None) -> None:
        """x_local: this rank's x entries (a CUDA tensor); y: its rows' result.

        Everything -- both all-reduce barriers, the window copy and the fused
        launch -- is ordered on one stream (`stream`, default torch's current
        one), which first waits for the caller's current stream (the work
        that produced x_local); the caller's stream then waits for it."""
        import contextlib

        import torch

        from .psc import BoundPlan

        b, e = self.ranges[self.rank]
        cuda = self.token.is_cuda
        ts = None
        if cuda and stream is not None:
            ts = stream if isinstance(stream, torch.cuda.Stream) else torch.cuda.ExternalStream(int(stream))
            ts.wait_stream(torch.cuda.current_stream())
        ctx = torch.cuda.stream(ts) if ts is not None else contextlib.nullcontext()
        with ctx:
            s = BoundPlan._stream(stream if ts is None else ts)
            self._sync()
            self.ipc.copy(self.window + 8 * b, x_local.data_ptr(), 8 * (e - b), s)
            self._sync()
            self.bound.spmv_peers(self.peers, self.window, y, s.value if ts is not None else stream)
        if ts is not None:
            torch.cuda.current_stream().wait_stream(ts)

    def close(self) -> None:
        for ptr in self.opened.values():
            self.ipc.close(ptr)
        self.opened = {}
        if self.window:
            self.ipc.free(self.window)
            self.window = 0
