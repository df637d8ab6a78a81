"""Config 4: split the gap of rows whose latest operand is in another piece into (operand published -> lane joined the
dense phase) and (joined -> row published). PSC_TRSV_TRACE=1 PSC_TRSV_TRACE_ROWS=2."""
import os, sys
sys.path.insert(0, "/root/repo")
os.environ["PSC_TRSV_TRACE"] = "1"; os.environ["PSC_TRSV_TRACE_ROWS"] = "2"
import ctypes as C
import numpy as np, torch
import paper_2111_12243_b200 as P
from paper_2111_12243_b200 import _capi
a = P.generate_config(4, 1.0)
plan = P.inspect(P.KernelKind.Sptrsv, a, 3, 8)
bound = P.BoundPlan(P.Executor(1, 0), plan, a)
b = torch.from_numpy(P.uniform_vector(a.n_rows, 1)).cuda(); x = torch.empty_like(b)
for _ in range(2): bound.sptrsv(b, x)
torch.cuda.synchronize()
n, nb = a.n_rows, bound.info()["work_units"]
buf = np.zeros(n + nb + 16, dtype=np.uint64)
_capi.lib().psc_bound_trace(bound._h, buf.ctypes.data_as(C.POINTER(C.c_uint64)), buf.size)
w = buf[:n]
pub = (w & np.uint64(0xFFFFFFFF)).astype(np.int64); join = (w >> np.uint64(32)).astype(np.int64)
dense = join != 0
M = 1 << 32
med = int(np.median(pub))
rel = lambda v: ((v - med + M // 2) % M) - M // 2  # low words, unwrapped around the median
pub = rel(pub); join = np.where(dense, rel(join), pub)
t0 = pub.min(); pub -= t0; join -= t0
print("rows via dense phase: %.1f%%; solve %.2f ms" % (100 * dense.mean(), pub.max() / 1e6))
ro, col = a.row_offsets, a.col_indices
last_dep = np.full(n, -1)
for r in range(n):
    k0, kd = ro[r], ro[r + 1] - 1
    if kd > k0:
        cs = col[k0:kd]; last_dep[r] = cs[np.argmax(pub[cs])]
has = last_dep >= 0
piece = np.zeros(n, dtype=np.int64); pid, start = -1, 0
for r in range(n):
    k0, kd = ro[r], ro[r + 1] - 1
    cont = r > 0 and kd > k0 and col[kd - 1] == r - 1
    if not cont or r - start >= 32:
        pid += 1; start = r
    piece[r] = pid
ld = np.maximum(last_dep, 0)
cross = has & (piece[ld] != piece)
g1 = join - pub[ld]; g2 = pub - join
sel = cross & dense
print("rows whose latest operand is in another piece: %d; operand -> join: median %.0f ns, p90 %.0f; join -> publish: median %.0f ns, p90 %.0f"
      % (sel.sum(), np.median(g1[sel]), np.percentile(g1[sel], 90), np.median(g2[sel]), np.percentile(g2[sel], 90)))
# critical path split
r = int(np.argmax(pub)); t_a = t_b = t_in = 0; hops = 0
while last_dep[r] >= 0:
    d = int(last_dep[r])
    if piece[d] != piece[r]:
        t_a += join[r] - pub[d]; t_b += pub[r] - join[r]; hops += 1
    else:
        t_in += pub[r] - pub[d]
    r = d
print("critical path: %d cross-piece hops: operand -> join %.2f ms, join -> publish %.2f ms; in-piece %.2f ms" % (hops, t_a / 1e6, t_b / 1e6, t_in / 1e6))
