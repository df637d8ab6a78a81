# config 2: tile size sweep of the record kernel (run under gpurun)
for R in ${ROWS:-10000 9600 9000}; do
  PSC_SPTRSV_BLOCK_ROWS=$R timeout 120 python bench.py --steps 50 --warmup 3 --no-cpu-baseline > gpurun_out/bs.json 2>&1
  python -c "import json; d=json.loads(open('gpurun_out/bs.json').read().strip().splitlines()[-1]); print('R=$R', 'kernel ms', round(d['roofline']['kernel_ms'],4), d['parity'], 'blocks', d['config']['bound']['work_units'])" || tail -3 gpurun_out/bs.json
done
