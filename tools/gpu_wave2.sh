#!/bin/bash
mkdir -p gpurun_out
for w in a; do
  PSC_TRSV_WAVE=$w timeout 600 python bench.py --config 2 --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/wave_c2_$w.jsonl 2> gpurun_out/wave_c2_$w.err; echo "rc=$?"
  python - <<PY
import json
for l in open("gpurun_out/wave_c2_$w.jsonl"):
    try: d=json.loads(l)
    except Exception: continue
    print("WAVE=$w", d.get("ms_per_step"), d.get("value"), d.get("roofline",{}).get("frac"))
PY
done
timeout 600 python tools/trace_sptrsv.py 2 1.0 > gpurun_out/wave_trace.log 2>&1; tail -25 gpurun_out/wave_trace.log
