# SpTRSV block-size sweep on config 2 (diagnostics; run under gpurun)
timeout 300 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout 200 python tools/trace_sptrsv.py 2 1.0 2>&1 | tail -14
for R in ${ROWS:-2048 4096 6757 10000 16384}; do
  echo "R=$R"; PSC_SPTRSV_BLOCK_ROWS=$R timeout 120 python bench.py --steps 30 --warmup 3 --no-cpu-baseline 2>&1 | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('ms', round(d['ms_per_step'],4), 'GF', round(d['value'],3), d['parity'], 'frac', round(d['roofline']['frac'],4), 'e2e_ms', round(d['e2e']['ms_per_step'],4))"
done
