"""Stage times of the GPU inspector vs the host inspector (needs a GPU).
Usage: python tools/insp_stages.py CONFIG [SCALE]"""
import os
import sys
import time

os.environ["PSC_INSPECT_TRACE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2111_12243_b200 as P  # noqa: E402

cfg = int(sys.argv[1])
scale = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
torch.cuda.init()
a = P.generate_config(cfg, scale)
kk = P.KernelKind.Spmv if cfg in (1, 3, 5) else P.KernelKind.Sptrsv
for rep in range(2):
    t0 = time.perf_counter()
    P.inspect(kk, a, 3, 8)
    t1 = time.perf_counter()
    P.inspect_device(kk, a, 3, 8)
    t2 = time.perf_counter()
    print(f"config {cfg} rep {rep}: host {t1 - t0:.3f} s, device {t2 - t1:.3f} s", flush=True)
