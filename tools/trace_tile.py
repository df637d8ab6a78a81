"""Step cadence of the level-synchronous solve on ONE block: the lower triangle
of a 7-point stencil on an nx x ny x nz grid (default 100 x 10 x 10, one
config-2 tile) bound as a single block. Compares with the whole config-2 run
to separate the loop's own cost from cross-block effects. Needs a GPU."""
import ctypes as C
import os
import sys

import numpy as np

if not os.environ.get("PSC_NO_TRACE"):
    os.environ["PSC_TRSV_TRACE"] = "1"
os.environ.setdefault("PSC_SPTRSV_BLOCK_ROWS", "12000")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2111_12243_b200 as P  # noqa: E402
from paper_2111_12243_b200 import _capi  # noqa: E402

nx, ny, nz = (int(v) for v in (sys.argv[1:4] if len(sys.argv) > 3 else (100, 10, 10)))
n = nx * ny * nz
rng = np.random.default_rng(7)
ro = [0]
ci, va = [], []
for r in range(n):
    x, y, z = r % nx, (r // nx) % ny, r // (nx * ny)
    for c in ([r - nx * ny] if z else []) + ([r - nx] if y else []) + ([r - 1] if x else []):
        ci.append(c)
        va.append(-1.0)
    ci.append(r)
    va.append(6.0 + 0.1 * rng.random())
    ro.append(len(ci))
a = P.CsrMatrix(n, n, np.array(ro, np.int32), np.array(ci, np.int32), np.array(va))
plan = P.inspect(P.KernelKind.Sptrsv, a, 3, 8)
bound = P.BoundPlan(P.Executor(1, 0), plan, a)
info = bound.info()
print("info", info)
b = torch.from_numpy(P.uniform_vector(n, 12)).cuda()
x = torch.empty_like(b)
for _ in range(3):
    bound.sptrsv(b, x)
torch.cuda.synchronize()
nb = info["work_units"]
if os.environ.get("PSC_NO_TRACE"):
    sys.exit(0)
buf = np.zeros(n + nb + 8, dtype=np.uint64)
_capi.lib().psc_bound_trace(bound._h, buf.ctypes.data_as(C.POINTER(C.c_uint64)), buf.size)
t = buf[:n].astype(np.int64)
t -= buf[n:n + nb].astype(np.int64).min()
r = np.arange(n)
lv = r % nx + (r // nx) % ny + r // (nx * ny)
lf = np.array([t[lv == l].max() for l in range(lv.max() + 1)])
d = np.diff(lf)
os.environ.pop("PSC_TRSV_TRACE", None)
b2 = P.BoundPlan(P.Executor(1, 0), plan, a)
ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for _ in range(3):
    b2.sptrsv(b, x)
ev0.record()
for _ in range(20):
    b2.sptrsv(b, x)
ev1.record()
torch.cuda.synchronize()
print(f"untraced solve {ev0.elapsed_time(ev1) / 20 * 1e3:.1f} us")
print(f"levels {lv.max() + 1}: first row {t.min()/1e3:.2f} us, last {t.max()/1e3:.2f} us, step median {np.median(d):.0f} ns mean {d.mean():.0f} ns")
