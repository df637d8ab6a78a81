#!/bin/bash
# Config 4 streaming solve: the solve tests, then the bench line (dense phase on / off).
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -x -q -m gpu -k "sptrsv or acceptance or configs or baselines or bound_device" > gpurun_out/c4_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/c4_pytest.log
tail -3 gpurun_out/c4_pytest.log
for d in 1 1 0; do
  PSC_TRSV_DENSE=$d timeout 900 python bench.py --config 4 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/c4_x.jsonl 2> gpurun_out/c4_x.err
  python - <<PY
import json
for l in open("gpurun_out/c4_x.jsonl"):
    try: d=json.loads(l)
    except Exception: continue
    print("DENSE=$d", d.get("ms_per_step"), d.get("roofline",{}).get("frac"))
PY
done
