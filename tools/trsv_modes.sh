# SpTRSV kernel variants on config 2 (diagnostics; run under gpurun)
timeout 300 python -m pytest tests -m gpu -x -q 2>&1 | tail -1
for LN in 1 0; do for M in 0 1; do
  echo "lean=$LN mode=$M"; PSC_TRSV_LEAN=$LN PSC_TRSV_MODE=$M timeout 120 python bench.py --steps 30 --warmup 3 --no-cpu-baseline 2>&1 | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('ms', round(d['ms_per_step'],4), 'GF', round(d['value'],3), d['parity'], 'frac', round(d['roofline']['frac'],4), 'e2e_ms', round(d['e2e']['ms_per_step'],4))"
done; done
