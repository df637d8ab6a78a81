"""Diagnostics: C2 solve timeline per plane (needs a GPU): when each z-plane's
first/last rows publish, and the in-line step time along x."""
import ctypes as C
import os
import sys

import numpy as np

os.environ["PSC_TRSV_TRACE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2111_12243_b200 as P  # noqa: E402
from paper_2111_12243_b200 import _capi  # noqa: E402

a = P.generate_config(2, 1.0)
plan = P.inspect(P.KernelKind.Sptrsv, a, 3, 8)
exe = P.Executor(1, 0)
bound = P.BoundPlan(exe, plan, a)
info = bound.info()
b = torch.from_numpy(P.uniform_vector(a.n_rows, 12)).cuda()
x = torch.empty_like(b)
for _ in range(3):
    bound.sptrsv(b, x)
torch.cuda.synchronize()
n, nb = a.n_rows, info["work_units"]
buf = np.zeros(n + nb + 8, dtype=np.uint64)
_capi.lib().psc_bound_trace(bound._h, buf.ctypes.data_as(C.POINTER(C.c_uint64)), buf.size)
t = buf[:n].astype(np.int64)
t -= t.min()
T = t.reshape(100, 100, 100)  # z, y, x
st = buf[n + nb:n + nb + 4].astype(float)
print(f"total {t.max()/1e3:.1f} us, blocks {nb}, block_rows {info['max_block_rows']}; rounds/warp {st[0]/max(st[2],1):.0f}, cycles/round {st[1]/max(st[0],1):.0f} (3 solves)")
for z in (0, 1, 2, 10, 50, 99):
    print(f"z={z:2d}: (0,0) {T[z,0,0]/1e3:8.1f}  (99,0) {T[z,0,99]/1e3:8.1f}  (0,99) {T[z,99,0]/1e3:8.1f}  "
          f"(99,99) {T[z,99,99]/1e3:8.1f} us")
dx = np.diff(T[:, :, :], axis=2)
print(f"x-step (same line) median {np.median(dx):.0f} ns, p90 {np.percentile(dx, 90):.0f} ns")
dy = T[:, 1:, :] - T[:, :-1, :]
print(f"y-lag median {np.median(dy):.0f} ns, p90 {np.percentile(dy, 90):.0f}")
dz = T[1:] - T[:-1]
print(f"z-lag median {np.median(dz):.0f} ns, p90 {np.percentile(dz, 90):.0f}")
