#!/bin/bash
mkdir -p gpurun_out
for ns in 0 20 50 100 200; do
  PSC_TRSV_POLL_NS=$ns timeout 600 python bench.py --config 2 --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/wave_c2_p$ns.jsonl 2> gpurun_out/wave_c2_p$ns.err
  python - <<PY
import json
for l in open("gpurun_out/wave_c2_p$ns.jsonl"):
    try: d=json.loads(l)
    except Exception: continue
    print("POLL_NS=$ns", d.get("ms_per_step"), d.get("roofline",{}).get("frac"), d.get("parity"))
PY
  PSC_TRSV_POLL_NS=$ns PSC_TRSV_TRACE_ROWS=0 timeout 600 python tools/trace_sptrsv.py 2 1.0 2>&1 | head -1
done
