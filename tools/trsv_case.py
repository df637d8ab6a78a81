"""One SpTRSV case with round statistics (diagnostics).
Usage (GPU): python tools/trsv_case.py CONFIG SCALE [THREADS] [BLOCK_ROWS] [REPS]
Env PSC_TRSV_* knobs apply. Prints time per solve, then (trace mode) warp
rounds, cycles per round and rows finished."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2111_12243_b200 as P  # noqa: E402
from paper_2111_12243_b200 import _capi  # noqa: E402

cfg, scale = int(sys.argv[1]), float(sys.argv[2])
if len(sys.argv) > 3:
    os.environ["PSC_TRSV_THREADS"] = sys.argv[3]
if len(sys.argv) > 4:
    os.environ["PSC_SPTRSV_BLOCK_ROWS"] = sys.argv[4]
reps = int(sys.argv[5]) if len(sys.argv) > 5 else 20
a = P.generate_config(cfg, scale)
plan = P.inspect(P.KernelKind.Sptrsv, a, 3, 8)
exe = P.Executor(1, 0)
bound = P.BoundPlan(exe, plan, a)
b = torch.from_numpy(P.uniform_vector(a.n_rows, 1)).cuda()
x = torch.empty_like(b)
for _ in range(3):
    bound.sptrsv(b, x)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(reps):
    bound.sptrsv(b, x)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / reps
info = bound.info()
levels = plan.counts().n_partitions
print(f"config {cfg} scale {scale}: n={a.n_rows} levels={levels} blocks={info['work_units']} "
      f"{ms*1e3:.1f} us/solve {ms*1e6/levels:.0f} ns/level", flush=True)
if os.environ.get("PSC_CASE_TRACE", "1") == "1":
    os.environ["PSC_TRSV_TRACE"] = "1"
    bound2 = P.BoundPlan(exe, plan, a)
    for _ in range(3):
        bound2.sptrsv(b, x)
    torch.cuda.synchronize()
    n, nb = a.n_rows, bound2.info()["work_units"]
    buf = np.zeros(n + nb + 8, dtype=np.uint64)
    got = _capi.lib().psc_bound_trace(bound2._h, buf.ctypes.data_as(_capi.C.POINTER(_capi.C.c_uint64)), buf.size)
    st = buf[n + nb:n + nb + 4].astype(float)
    print(f"  warps {st[2]/3:.0f} rounds/warp {st[0]/max(st[2],1):.0f} cycles/round {st[1]/max(st[0],1):.0f} "
          f"rows/warp {st[3]/max(st[2],1):.0f}", flush=True)
