"""Diagnostics: one pinned-buffer host-path SpTRSV call on a small config 2,
checked against the device path. Usage (GPU): python tools/host_path_probe.py [SCALE]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2111_12243_b200 as P  # noqa: E402

scale = float(sys.argv[1]) if len(sys.argv) > 1 else 0.03
a = P.generate_config(2, scale)
plan = P.inspect(P.KernelKind.Sptrsv, a, 3, 8)
bound = P.BoundPlan(P.Executor(1, 0), plan, a)
print("bound", bound.info(), flush=True)
bh = torch.from_numpy(P.uniform_vector(a.n_rows, 1)).pin_memory()
xh = torch.full((a.n_rows,), float("nan"), dtype=torch.float64).pin_memory()
bd = bh.cuda()
xd = torch.empty_like(bd)
bound.sptrsv(bd, xd)
torch.cuda.synchronize()
print("device path done", flush=True)
t0 = time.time()
bound.sptrsv_host(bh.numpy(), xh.numpy())
print("enqueued", time.time() - t0, flush=True)
torch.cuda.synchronize()
print("host path done", time.time() - t0, np.array_equal(xh.numpy().view(np.int64), xd.cpu().numpy().view(np.int64)),
      flush=True)
