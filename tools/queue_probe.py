"""Diagnostics: per-row latency of the unit-queue solve kernel in isolation
(one dense lower triangle = one chain = one warp). Usage (GPU):
python tools/queue_probe.py [N]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2111_12243_b200 as P  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 300
rng = np.random.default_rng(0)
ent = []
for r in range(n):
    for c in range(r):
        ent.append((r, c, float(rng.uniform(-1, 1)) / n))
    ent.append((r, r, 2.0))
a = P.csr_from_triplets(n, n, ent)
plan = P.inspect(P.KernelKind.Sptrsv, a, 3, 8)
bound = P.BoundPlan(P.Executor(1, 0), plan, a)
b = torch.from_numpy(P.uniform_vector(n, 1)).cuda()
x = torch.empty_like(b)
for _ in range(3):
    bound.sptrsv(b, x)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(20):
    bound.sptrsv(b, x)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 20
print(f"dense triangle n={n} (mean row {n / 2:.0f} entries, segments/row ~{plan.counts().n_codelets / n:.1f}): "
      f"{ms * 1e3:.1f} us, {ms * 1e6 / n:.0f} ns/row", flush=True)
