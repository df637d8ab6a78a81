"""Diagnostics for config 4 (supernodal SpTRSV): per-row publish times from
the warp-per-unit kernel (PSC_TRSV_TRACE=1); splits row-to-row time into the
in-chain step (row r-1 of the same unit) and waits on other rows.
Usage (GPU): python tools/trace_c4.py [SCALE]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["PSC_TRSV_TRACE"] = "1"
import ctypes as C  # noqa: E402

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2111_12243_b200 as P  # noqa: E402
from paper_2111_12243_b200 import _capi  # noqa: E402

scale = float(sys.argv[1]) if len(sys.argv) > 1 else 1.0
a = P.generate_config(4, scale)
plan = P.inspect(P.KernelKind.Sptrsv, a, 3, 8)
bound = P.BoundPlan(P.Executor(1, 0), plan, a)
b = torch.from_numpy(P.uniform_vector(a.n_rows, 1)).cuda()
x = torch.empty_like(b)
for _ in range(2):
    bound.sptrsv(b, x)
torch.cuda.synchronize()
n, nb = a.n_rows, bound.info()["work_units"]
buf = np.zeros(n + nb + 16, dtype=np.uint64)
_capi.lib().psc_bound_trace(bound._h, buf.ctypes.data_as(C.POINTER(C.c_uint64)), buf.size)
t = buf[:n].astype(np.int64)
t -= t.min()
ro, col = a.row_offsets, a.col_indices
# the latest-finishing operand of every row, and whether it is the row above
last_dep = np.full(n, -1)
for r in range(n):
    k0, kd = ro[r], ro[r + 1] - 1
    if kd > k0:
        cs = col[k0:kd]
        last_dep[r] = cs[np.argmax(t[cs])]
has = last_dep >= 0
gap = np.where(has, t - t[np.maximum(last_dep, 0)], 0)
chain = has & (last_dep == np.arange(n) - 1)
print(f"solve {t.max() / 1e6:.2f} ms, rows {n}")
print(f"gap after the latest operand: median {np.median(gap[has]):.0f} ns, p90 {np.percentile(gap[has], 90):.0f} ns")
print(f"  latest operand = row above (chain): {chain.mean():.2%}, median {np.median(gap[chain]):.0f} ns")
print(f"  latest operand elsewhere: median {np.median(gap[has & ~chain]):.0f} ns")
# critical path: follow latest operands back from the last-finishing row
r = int(np.argmax(t))
steps, in_chain = 0, 0
while last_dep[r] >= 0:
    in_chain += last_dep[r] == r - 1
    r = int(last_dep[r])
    steps += 1
print(f"critical path: {steps} hops, {in_chain} of them in-chain; mean {t.max() / max(steps, 1):.0f} ns per hop")
ln = (ro[1:] - ro[:-1]) - 1
for lo, hi in ((0, 64), (64, 128), (128, 256), (256, 512), (512, 10 ** 9)):
    sel = chain & (ln >= lo) & (ln < hi)
    if sel.any():
        print(f"  in-chain rows with {lo}-{hi} entries: {sel.sum()} rows, median {np.median(gap[sel]):.0f} ns")
print(f"row length: median {np.median(ln):.0f}, p99 {np.percentile(ln, 99):.0f}, max {ln.max()}")
# streaming kernel pieces: chain units cut every 32 rows
piece = np.zeros(n, dtype=np.int64)
pid, start = -1, 0
for r in range(n):
    k0, kd = ro[r], ro[r + 1] - 1
    cont = r > 0 and kd > k0 and col[kd - 1] == r - 1
    if not cont or r - start >= 32:
        pid += 1
        start = r if not cont or r - start >= 32 else start
        if not cont:
            start = r
    piece[r] = pid
same = has & (piece[np.maximum(last_dep, 0)] == piece)
print(f"latest operand in the same piece: {same.mean():.2%} (median gap {np.median(gap[same]):.0f} ns); "
      f"in another piece: {(has & ~same).mean():.2%} (median gap {np.median(gap[has & ~same]):.0f} ns)")
r = int(np.argmax(t))
hops_same = hops_other = 0
t_same = t_other = 0
while last_dep[r] >= 0:
    d = int(last_dep[r])
    if piece[d] == piece[r]:
        hops_same += 1
        t_same += t[r] - t[d]
    else:
        hops_other += 1
        t_other += t[r] - t[d]
    r = d
print(f"critical path: {hops_same} in-piece hops ({t_same / 1e6:.2f} ms, {t_same / max(hops_same, 1):.0f} ns each), "
      f"{hops_other} cross-piece hops ({t_other / 1e6:.2f} ms, {t_other / max(hops_other, 1):.0f} ns each)")
st4 = buf[n:n + 9].astype(np.float64)
print(f"triangle phases: {st4[7] / max(st4[4], 1):.0f} cycles each, {st4[7] / max(st4[8], 1):.0f} cycles per column")
print(f"pieces (2 solves): {st4[6]:.0f}; finished by the triangle phase {st4[4]:.0f}, of them with the previous piece in the window {st4[5]:.0f}")  # streaming kernel: rounds with / without L2 operand loads, and their cycles
if st4[0] + st4[2] > 0:
    print(f"stream rounds (2 solves, all warps): with L2 loads {st4[0]:.0f} ({st4[1] / max(st4[0], 1):.0f} cycles each), "
          f"smem only {st4[2]:.0f} ({st4[3] / max(st4[2], 1):.0f} cycles each)")
