# config 1: CTA size of the thread-per-row kernel (run under gpurun)
b() { timeout 300 python bench.py --config 1 --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/r.json 2>&1; python -c "
import json; d=json.loads(open('gpurun_out/r.json').read().strip().splitlines()[-1]); print('$1', d['parity'], 'kernel us', round(d['roofline']['kernel_ms']*1e3,2), 'frac', round(d['roofline']['frac'],3))"; }
for rb in 256 128 512 64; do PSC_ROWK_BLOCK=$rb b block$rb; done
