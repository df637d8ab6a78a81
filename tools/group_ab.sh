# SpMV row groups on config 3 (run under gpurun)
timeout 900 python -m pytest tests -m gpu -q -x -k "spmv or configs or acceptance or edge or shard" > gpurun_out/g_pytest.log 2>&1; tail -1 gpurun_out/g_pytest.log
b() { timeout 600 python bench.py --config 3 --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/g.json 2>&1; python -c "
import json; d=json.loads(open('gpurun_out/g.json').read().strip().splitlines()[-1]); print('$1', d['parity'], 'kernel ms', round(d['roofline']['kernel_ms'],4), 'frac', round(d['roofline']['frac'],3), 'e2e', round(d['e2e']['ms_per_step'],3))" || tail -5 gpurun_out/g.json; }
b overlap; b overlap_again
