# config 2: record-kernel spin back-off (run under gpurun)
for sp in 0 20 50 100; do PSC_TRSV_SPIN=$sp timeout 300 python bench.py --steps 100 --warmup 5 --no-cpu-baseline > gpurun_out/sp.json 2>&1; python -c "
import json; d=json.loads(open('gpurun_out/sp.json').read().strip().splitlines()[-1]); print('spin=$sp', d['parity'], 'kernel ms', round(d['roofline']['kernel_ms'],4))"; done
