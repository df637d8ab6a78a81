"""Summarise warp-stall samples per SASS instruction from `ncu --page source
--csv --print-source sass` output. Usage: python tools/ncu_stalls.py FILE.csv [TOP]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top_n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
hdr = rows[1]
data = rows[2:]
i_s = hdr.index("Warp Stall Sampling (All Samples)")
i_e = hdr.index("Instructions Executed")
reasons = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
ri = [hdr.index(h) for h in reasons]
tot = sum(float(r[i_s] or 0) for r in data) or 1.0
print("total samples", tot, "warp instructions", sum(int(r[i_e] or 0) for r in data))
agg = {h: sum(float(r[i] or 0) for r in data) for h, i in zip(reasons, ri)}
print({k: round(v / tot * 100, 1) for k, v in sorted(agg.items(), key=lambda kv: -kv[1])[:8]})
idx = sorted(range(len(data)), key=lambda k: -float(data[k][i_s] or 0))[:top_n]
for k in sorted(idx):
    r = data[k]
    top = max(zip(reasons, ri), key=lambda hi: float(r[hi[1]] or 0))[0]
    print(f"{k:5d} {float(r[i_s]) / tot * 100:5.1f}% ex={r[i_e]:>7s} {top:18s} {r[1][:80]}")
