#!/bin/bash
# Config 4 streaming solve: the bench line (dense phase on / off).
mkdir -p gpurun_out
for d in 1 1 0; do
  PSC_TRSV_DENSE=$d timeout 900 python bench.py --config 4 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/c4_x.jsonl 2> gpurun_out/c4_x.err
  python - <<PY
import json
for l in open("gpurun_out/c4_x.jsonl"):
    try: d=json.loads(l)
    except Exception: continue
    print("DENSE=$d", d.get("ms_per_step"), d.get("roofline",{}).get("frac"), d.get("clocks"))
PY
done
