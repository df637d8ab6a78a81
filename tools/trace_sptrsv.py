"""Diagnostics: per-row publish times of one SpTRSV solve, grouped by
dependency level (needs a GPU). Usage: python tools/trace_sptrsv.py [config] [scale]"""
import ctypes as C
import os
import sys

import numpy as np

os.environ["PSC_TRSV_TRACE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2111_12243_b200 as P  # noqa: E402
from paper_2111_12243_b200 import _capi  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
scale = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
a = P.generate_config(cfg, scale)
plan = P.inspect(P.KernelKind.Sptrsv, a, 3, 8)
exe = P.Executor(1, 0)
bound = P.BoundPlan(exe, plan, a)
info = bound.info()
b = torch.from_numpy(P.uniform_vector(a.n_rows, 12)).cuda()
x = torch.empty_like(b)
for _ in range(3):
    bound.sptrsv(b, x)
torch.cuda.synchronize()
n = a.n_rows
nb = info["work_units"]
buf = np.zeros(n + nb + 8, dtype=np.uint64)
got = _capi.lib().psc_bound_trace(bound._h, buf.ctypes.data_as(C.POINTER(C.c_uint64)), buf.size)
assert got == n + nb + 8, got
stats = buf[n + nb:n + nb + 4].astype(np.float64); buf = buf[:n + nb]
rounds = stats[0]
print(f'warps {stats[2]:.0f} rounds/warp {stats[0]/max(stats[2],1):.0f} cycles/round {stats[1]/max(stats[0],1):.0f} rows {stats[3]:.0f} (3 solves accumulated)')
t_rows = buf[:n].astype(np.int64)
t_arm = buf[n:].astype(np.int64)
t0 = t_arm.min()
t_rows -= t0
t_arm -= t0
# dependency levels
level = np.zeros(n, dtype=np.int64)
ro, ci = a.row_offsets, a.col_indices
for r in range(n):
    k0, k1 = ro[r], ro[r + 1] - 1
    if k1 > k0:
        level[r] = level[ci[k0:k1]].max() + 1
L = level.max() + 1
print(f"n={n} levels={L} blocks={nb} block_rows={info.get('max_block_rows', info.get('passes_or_block_rows', 10000))}")
print(f"arm times (us): min {t_arm.min()/1e3:.1f} max {t_arm.max()/1e3:.1f}")
print(f"total (last publish) {t_rows.max()/1e3:.1f} us; warp rounds (sum over warps, 3 solves) {rounds}")
lv_max = np.zeros(L)
for l in range(L):
    lv_max[l] = t_rows[level == l].max()
step = np.diff(lv_max)
print("per-level finish (us) at levels 0,10,50,100,150,200,250,last:",
      [round(lv_max[i] / 1e3, 1) for i in (0, 10, 50, 100, 150, 200, 250, L - 1) if i < L])
print(f"per-level step: median {np.median(step)/1e3:.2f} us, mean {step.mean()/1e3:.2f} us, max {step.max()/1e3:.1f} us")
blk = np.arange(n) // info.get("max_block_rows", info.get("passes_or_block_rows", 10000))
for k in list(range(0, nb, max(1, nb // 8)))[:10]:
    m = blk == k
    print(f"block {k}: rows finish {t_rows[m].min()/1e3:.1f}..{t_rows[m].max()/1e3:.1f} us, levels {level[m].min()}..{level[m].max()}")
if cfg == 2 and scale == 1.0:  # per-line cadence inside the first planes (rows r = x + 100 y + 10000 z)
    N = 100
    for z in (0, 1, 50):
        t = t_rows[z * N * N:(z + 1) * N * N].reshape(N, N)  # [y][x]
        first = t[:, 0] / 1e3
        step_x = np.median(np.diff(t, axis=1), axis=1)  # per line: median time between consecutive rows
        print(f"plane z={z}: line start (us) y=0,1,2,31,32,63,64,99: {[round(first[i], 2) for i in (0, 1, 2, 31, 32, 63, 64, 99)]}")
        print(f"  median row step along x (ns) y=0,1,31,32,99: {[int(step_x[i]) for i in (0, 1, 31, 32, 99)]}; line end (us) y=0,99: {round(t[0,-1]/1e3,2)}, {round(t[99,-1]/1e3,2)}")
