#!/bin/bash
mkdir -p gpurun_out
for mb in 1 8 1 8; do
  PSC_RUN_MINB=$mb timeout 600 python bench.py --config 1 --steps 50 --warmup 10 --no-cpu-baseline > gpurun_out/c1_mb$mb.jsonl 2> gpurun_out/c1_mb$mb.err
  python - <<PY
import json
for l in open("gpurun_out/c1_mb$mb.jsonl"):
    try: d=json.loads(l)
    except Exception: continue
    print("MINB=$mb", d.get("ms_per_step"), d.get("roofline",{}).get("frac"))
PY
done
