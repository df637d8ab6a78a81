# SpMV configs 1/3/5 (run under gpurun)
timeout 400 python -m pytest tests -m gpu -q -x 2>&1 | tail -2 | head -1
for c in 1 3 5; do timeout 400 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c$c.json 2>&1; python -c "
import json; d=json.loads(open('gpurun_out/bench_c$c.json').read().strip().splitlines()[-1])
print($c, 'ms', round(d['ms_per_step'],4), 'GF', round(d['value'],1), d['parity'], 'frac', round(d['roofline']['frac'],3), 'GB/s', round(d['roofline']['achieved']), 'e2e ms', round(d['e2e']['ms_per_step'],3), 'launches', d['gpu_launches'])"; done
