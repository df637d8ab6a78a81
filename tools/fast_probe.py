"""A/B of SpMV bind variants on one config (GPU box): parity vs fast mode
with environment knobs read at bind time. Prints one line per variant:
median ms over cold-L2 reps, fraction of the HBM roofline, normwise error
against the parity result (itself bitwise the reference executor's).

    python tools/fast_probe.py --config 5 --variants 'fast:PSC_FAST_SPLIT_BYTES=80000000' ...
"""
import argparse
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2111_12243_b200 as P  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=5)
ap.add_argument("--scale", type=float, default=1.0)
ap.add_argument("--reps", type=int, default=20)
ap.add_argument("--variants", nargs="+", default=["parity:", "fast:"])
args = ap.parse_args()

peak = json.load(open(os.path.join(os.path.dirname(__file__), "..", "MEASURED_PEAKS.json")))["hbm_gbs"]
t0 = time.time()
a = P.generate_config(args.config, args.scale)
plan = P.inspect(P.KernelKind.Spmv, a, 3, 8)
print(f"config {args.config}: n={a.n_rows} nnz={a.nnz()} gen+inspect {time.time() - t0:.1f}s", flush=True)
exe = P.Executor(1, 0)
x = torch.from_numpy(P.uniform_vector(a.n_cols, 10 + args.config)).cuda()
l2 = torch.cuda.get_device_properties(0).L2_cache_size
fl1 = torch.empty(2 * l2 // 4, dtype=torch.float32, device="cuda")
fl2 = torch.ones(2 * l2 // 4, dtype=torch.float32, device="cuda")
sink = torch.empty((), dtype=torch.float32, device="cuda")
ref = None
for v in args.variants:
    mode_s, _, env_s = v.partition(":")
    env = dict(kv.split("=", 1) for kv in env_s.split(",") if kv)
    old = {k: os.environ.get(k) for k in env}
    os.environ.update(env)
    t0 = time.time()
    b = P.BoundPlan(exe, plan, a, mode=1 if mode_s == "fast" else 0)
    bind_s = time.time() - t0
    for k, o in old.items():
        if o is None:
            del os.environ[k]
        else:
            os.environ[k] = o
    y = torch.empty(a.n_rows, dtype=torch.float64, device="cuda")
    ms = []
    for i in range(args.reps + 3):
        fl1.zero_()
        torch.sum(fl2, 0, out=sink)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        b.spmv(x, y)
        e1.record()
        torch.cuda.synchronize()
        if i >= 3:
            ms.append(e0.elapsed_time(e1))
    yh = y.cpu().numpy()
    if ref is None:
        ref = yh
    err = float(np.max(np.abs(yh - ref)) / max(np.max(np.abs(ref)), 1e-300))
    bits = bool(np.array_equal(yh.view(np.int64), ref.view(np.int64)))
    med = float(np.median(ms))
    ab = b.info()["algorithmic_bytes"]
    print(f"{v:60s} {med:8.4f} ms  frac {ab / med / 1e6 / peak:.3f}  min {min(ms):.4f}  normwise {err:.2e} "
          f"bitwise {bits}  launches {b.launches()}  bind {bind_s:.1f}s", flush=True)
    b.close()
    del y
