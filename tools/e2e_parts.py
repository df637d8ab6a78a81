"""Diagnostics: time the parts of the host-buffer SpTRSV step on one stream.
Usage (GPU): python tools/e2e_parts.py [CONFIG] [SCALE]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2111_12243_b200 as P  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
scale = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
a = P.generate_config(cfg, scale)
plan = P.inspect(P.KernelKind.Sptrsv, a, 3, 8)
bound = P.BoundPlan(P.Executor(1, 0), plan, a)
n = a.n_rows
bh = torch.from_numpy(P.uniform_vector(n, 1)).pin_memory()
xh = torch.empty(n, dtype=torch.float64).pin_memory()
xpage = np.empty(n)
bd = bh.cuda()
xd = torch.empty_like(bd)
s = torch.cuda.current_stream()


def timeit(label, fn, reps=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    print(f"{label:44s} {e0.elapsed_time(e1) / reps * 1e3:9.1f} us", flush=True)


timeit("H2D 8 B/row (pinned)", lambda: bd.copy_(bh, non_blocking=True))
timeit("D2H 8 B/row (pinned)", lambda: xh.copy_(xd, non_blocking=True))
timeit("solve, device buffers", lambda: bound.sptrsv(bd, xd))
timeit("host path, pinned b and x (overlapped)", lambda: bound.sptrsv_host(bh.numpy(), xh.numpy()))
timeit("host path, pinned b, pageable x", lambda: bound.sptrsv_host(bh.numpy(), xpage))

import time  # noqa: E402

for label, fn in (("host path, pinned b and x (overlapped)", lambda: bound.sptrsv_host(bh.numpy(), xh.numpy())),):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(20):
        fn()
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    print(f"{label}: host enqueue {(t1 - t0) / 20 * 1e6:.1f} us/call, wall {(t2 - t0) / 20 * 1e6:.1f} us/call")
