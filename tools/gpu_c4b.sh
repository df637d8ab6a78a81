#!/bin/bash
# Config 4: buffers per L2 round (PSC_TRSV_BURST) A/B and the critical-path trace.
mkdir -p gpurun_out
for b in 8 16 64 8 16; do
  PSC_TRSV_BURST=$b timeout 900 python bench.py --config 4 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/c4_burst$b.jsonl 2> gpurun_out/c4_burst$b.err
  python - <<PY
import json
for l in open("gpurun_out/c4_burst$b.jsonl"):
    try: d=json.loads(l)
    except Exception: continue
    print("BURST=$b", d.get("ms_per_step"), d.get("roofline",{}).get("frac"))
PY
done
timeout 900 python tools/trace_c4.py 1.0 2>&1 | tee gpurun_out/c4_trace_burst8.log | tail -8
