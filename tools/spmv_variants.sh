# SpMV kernel variants x configs (run under gpurun)
for V in 0 1 2 3 4; do for c in 1 3 5; do PSC_SPMV_VARIANT=$V timeout 400 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/bench_v${V}_c$c.json 2>&1; python -c "
import json; d=json.loads(open("gpurun_out/bench_v${V}_c$c.json").read().strip().splitlines()[-1])
print('v$V', $c, 'ms', round(d['ms_per_step'],4), 'GF', round(d['value'],1), d['parity'], 'frac', round(d['roofline']['frac'],3))"; done; done
