"""Single-lane chain (bidiagonal, one block) solve, for per-row latency
analysis under ncu. Usage (GPU): python tools/trsv_chain.py [N] [REPS]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2111_12243_b200 as P  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
os.environ.setdefault("PSC_SPTRSV_BLOCK_ROWS", str(n))
os.environ.setdefault("PSC_TRSV_THREADS", "64")
a = P.banded(n, 1, True)
for v in range(a.nnz()):
    a.values[v] = 1.0 if a.col_indices[v] == np.searchsorted(a.row_offsets, v, "right") - 1 else 0.5
plan = P.inspect(P.KernelKind.Sptrsv, a, 3, 8)
bound = P.BoundPlan(P.Executor(1, 0), plan, a)
b = torch.from_numpy(P.uniform_vector(n, 1)).cuda()
x = torch.empty_like(b)
for _ in range(2):
    bound.sptrsv(b, x)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(reps):
    bound.sptrsv(b, x)
e1.record()
torch.cuda.synchronize()
print(f"chain n={n}: {e0.elapsed_time(e1) / reps * 1e6 / n:.1f} ns/row", flush=True)
