# column-split SpMV on config 5 (run under gpurun)
timeout 900 python -m pytest tests/test_gpu_edges.py -m gpu -q -x -k "split" > gpurun_out/sp_pytest.log 2>&1; tail -3 gpurun_out/sp_pytest.log
b() { timeout 900 python bench.py --config 5 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/sp.json 2>&1; python -c "
import json; d=json.loads(open('gpurun_out/sp.json').read().strip().splitlines()[-1]); print('$1', d['parity'], 'kernel ms', round(d['roofline']['kernel_ms'],3), 'frac', round(d['roofline']['frac'],3), 'launches', d['gpu_launches'], 'e2e ms', round(d['e2e']['ms_per_step'],3))" || tail -5 gpurun_out/sp.json; }
b default
