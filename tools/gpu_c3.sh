#!/bin/bash
# Config 3 (row groups): shifted group templates on / off, after the SpMV tests.
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -x -q -m gpu -k "spmv or acceptance or configs or bound_device or fast or groups" > gpurun_out/c3_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/c3_pytest.log
tail -3 gpurun_out/c3_pytest.log
for sg in 1 0 1 0; do
  PSC_SPMV_GROUP_SHIFT=$sg timeout 900 python bench.py --config 3 --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/c3_x.jsonl 2> gpurun_out/c3_x.err
  python - <<PY
import json
for l in open("gpurun_out/c3_x.jsonl"):
    try: d=json.loads(l)
    except Exception: continue
    print("GROUP_SHIFT=$sg", d.get("ms_per_step"), d.get("roofline",{}).get("frac"))
PY
done
