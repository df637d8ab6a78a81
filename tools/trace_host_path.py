"""Diagnostics: per-row finish times of the SpTRSV solve through the pinned
host path (b streamed in during the solve, x shipped out), config 2.
Usage (GPU): python tools/trace_host_path.py"""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["PSC_TRSV_TRACE"] = "1"
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2111_12243_b200 as P  # noqa: E402
from paper_2111_12243_b200 import _capi  # noqa: E402

a = P.generate_config(2, 1.0)
plan = P.inspect(P.KernelKind.Sptrsv, a, 3, 8)
bound = P.BoundPlan(P.Executor(1, 0), plan, a)
n, nb = a.n_rows, bound.info()["work_units"]
bh = torch.from_numpy(P.uniform_vector(n, 1)).pin_memory()
xh = torch.empty(n, dtype=torch.float64).pin_memory()
for mode in ("device", "host"):
    for _ in range(3):
        if mode == "host":
            bound.sptrsv_host(bh.numpy(), xh.numpy())
        else:
            bd, xd = bh.cuda(), torch.empty(n, dtype=torch.float64, device="cuda")
            torch.cuda.synchronize()
            bound.sptrsv(bd, xd)
    torch.cuda.synchronize()
    buf = np.zeros(n + nb + 8, dtype=np.uint64)
    _capi.lib().psc_bound_trace(bound._h, buf.ctypes.data_as(C.POINTER(C.c_uint64)), buf.size)
    t = buf[:n].astype(np.int64)
    arm = buf[n:n + nb].astype(np.int64)
    t0 = arm.min()
    t = (t - t0) / 1e3
    T = t.reshape(100, 100, 100)
    print(f"[{mode}] last row {t.max():.1f} us after the first block armed")
    for z in (0, 12, 25, 50, 75, 87, 99):
        print(f"  z={z:2d}: (0,0) {T[z, 0, 0]:7.1f}  (99,99) {T[z, 99, 99]:7.1f} us")
