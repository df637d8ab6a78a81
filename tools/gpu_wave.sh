#!/bin/bash
# Wavefront record kernel: solve tests, config 2 timing, loop counters.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu -k "${WAVE_TESTS:-sptrsv or acceptance or configs or edges or baselines or bound_device}" > gpurun_out/wave_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/wave_pytest.log
tail -5 gpurun_out/wave_pytest.log
for w in ${WAVE_MODES:-a}; do
  PSC_TRSV_WAVE=$w timeout 600 python bench.py --config 2 --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/wave_c2_$w.jsonl 2> gpurun_out/wave_c2_$w.err; echo "rc=$?"
  python - <<PY
import json
for l in open("gpurun_out/wave_c2_$w.jsonl"):
    try: d=json.loads(l)
    except Exception: continue
    print("WAVE=$w", d.get("ms_per_step"), d.get("value"), d.get("roofline",{}).get("frac"))
PY
done
PSC_TRSV_TRACE_ROWS=0 PSC_TRSV_WAVE=a timeout 600 python tools/trace_sptrsv.py 2 1.0 > gpurun_out/wave_trace0.log 2>&1; head -2 gpurun_out/wave_trace0.log
