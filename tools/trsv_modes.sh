# SpTRSV lean kernel: burst x mode (diagnostics; run under gpurun)
timeout 300 python -m pytest tests/test_gpu_parity.py -q -x 2>&1 | tail -1
for B in 1 2 4 8; do for M in 1 0; do
  echo "burst=$B mode=$M"; PSC_TRSV_BURST=$B PSC_TRSV_MODE=$M timeout 120 python bench.py --steps 30 --warmup 3 --no-cpu-baseline 2>&1 | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('ms', round(d['ms_per_step'],4), 'GF', round(d['value'],3), d['parity'], 'frac', round(d['roofline']['frac'],4))"
done; done
PSC_TRSV_BURST=4 PSC_TRSV_MODE=1 timeout 100 python tools/trace_planes.py
