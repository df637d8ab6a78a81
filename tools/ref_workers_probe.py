"""Diagnostics: does the reference executor survive multi-worker SpTRSV on
config 2, and how fast is it? Each trial runs in a subprocess (the
reference's pool race can SEGV). Usage: python tools/ref_workers_probe.py"""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHILD = r"""
import sys, numpy as np
sys.path.insert(0, %r)
import paper_2111_12243_b200 as P
from oracle.oracle import Ref
w = int(sys.argv[1])
a = P.generate_config(2, 1.0)
rc = Ref.csr(a.view())
plan, _ = Ref.time_inspect(1, rc, 3, 8)
b = P.uniform_vector(a.n_rows, 12)
times, x = Ref.time_sptrsv(plan, rc, b, w, 2, 5)
print("workers", w, "median ms", float(np.median(times)) * 1e3, flush=True)
""" % ROOT

for w in (1, 4, 16, os.cpu_count()):
    ok = 0
    for trial in range(3):
        p = subprocess.run([sys.executable, "-c", CHILD, str(w)], capture_output=True, text=True, timeout=300)
        if p.returncode == 0:
            ok += 1
            last = p.stdout.strip().splitlines()[-1]
        else:
            last = f"rc={p.returncode} {p.stderr.strip().splitlines()[-1] if p.stderr.strip() else ''}"
    print(f"workers={w}: {ok}/3 ok; {last}", flush=True)
