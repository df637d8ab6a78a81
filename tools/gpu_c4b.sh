#!/bin/bash
# Config 4: buffers per L2 round (PSC_TRSV_BURST) A/B, after the solve tests with bursts on.
mkdir -p gpurun_out
PSC_TRSV_BURST=4 timeout 1200 python -m pytest tests -x -q -m gpu -k "sptrsv or acceptance or configs or baselines or bound_device" > gpurun_out/c4b_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/c4b_pytest.log
tail -3 gpurun_out/c4b_pytest.log
for b in 1 2 4 8 1 4; do
  PSC_TRSV_BURST=$b timeout 900 python bench.py --config 4 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/c4_burst$b.jsonl 2> gpurun_out/c4_burst$b.err
  python - <<PY
import json
for l in open("gpurun_out/c4_burst$b.jsonl"):
    try: d=json.loads(l)
    except Exception: continue
    print("BURST=$b", d.get("ms_per_step"), d.get("roofline",{}).get("frac"))
PY
done
