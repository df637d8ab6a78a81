#!/bin/bash
mkdir -p gpurun_out
for cfg in "1 4" "2 4" "4 4" "2 8" "4 8"; do
  set -- $cfg
  PSC_TRSV_BURST=$1 PSC_TRSV_STREAM_WARPS=$2 timeout 900 python bench.py --config 4 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/c4_x.jsonl 2> gpurun_out/c4_x.err
  python - <<PY
import json
for l in open("gpurun_out/c4_x.jsonl"):
    try: d=json.loads(l)
    except Exception: continue
    print("BURST=$1 WARPS=$2", d.get("ms_per_step"), d.get("roofline",{}).get("frac"))
PY
done
timeout 900 python tools/trace_c4.py 1.0 2>&1 | tee gpurun_out/c4_trace_incr.log | tail -7
