#!/bin/bash
# Config 1 (thread-per-row SpMV): shifted-run items on and off, and the SpMV tests.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu -k "spmv or acceptance or configs or bound_device or fast" > gpurun_out/c1_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/c1_pytest.log
tail -5 gpurun_out/c1_pytest.log
for runs in 1 0; do
  PSC_SPMV_RUNS=$runs timeout 600 python bench.py --config 1 --steps 50 --warmup 10 --no-cpu-baseline > gpurun_out/c1_runs$runs.jsonl 2> gpurun_out/c1_runs$runs.err; echo "rc=$?"
  python - <<PY
import json
for l in open("gpurun_out/c1_runs$runs.jsonl"):
    try: d=json.loads(l)
    except Exception: continue
    print("RUNS=$runs", d.get("ms_per_step"), d.get("value"), d.get("roofline",{}).get("frac"), d.get("bound"))
PY
done
