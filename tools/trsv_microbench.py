"""Diagnostics: per-level latency of the solve kernel on pure chains
(bidiagonal: one row per level) and on small single-block 3-D grids.
Usage (GPU): python tools/trsv_microbench.py"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2111_12243_b200 as P  # noqa: E402


def run(a, label, reps=20):
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
    levels = plan.counts().n_partitions
    info = bound.info()
    print(f"{label:38s} n={a.n_rows:8d} levels={levels:6d} blocks={info['work_units']:4d} "
          f"{ms*1e3:9.1f} us  {ms*1e6/levels:8.1f} ns/level", flush=True)


chain = P.banded(8192, 1, True)
for v in range(chain.nnz()):
    chain.values[v] = 1.0 if chain.col_indices[v] == np.searchsorted(chain.row_offsets, v, "right") - 1 else 0.5
for T in (64, 128, 512):
    os.environ["PSC_TRSV_THREADS"] = str(T)
    os.environ["PSC_SPTRSV_BLOCK_ROWS"] = "8192"
    run(chain, f"bidiagonal 8192, 1 block, T={T}")
for R in (1024, 4096):
    os.environ["PSC_TRSV_THREADS"] = "512"
    os.environ["PSC_SPTRSV_BLOCK_ROWS"] = str(R)
    run(chain, f"bidiagonal 8192, blocks of {R}, T=512")
os.environ["PSC_SPTRSV_BLOCK_ROWS"] = "12000"
for T in (128, 512):
    os.environ["PSC_TRSV_THREADS"] = str(T)
    run(P.generate_config(2, 0.01), f"3D 7pt 22^3 one block T={T}")
os.environ.pop("PSC_SPTRSV_BLOCK_ROWS")
os.environ["PSC_TRSV_THREADS"] = "512"
run(P.generate_config(2, 1.0), "config 2 default")
