# config 1 SpMV: rows per thread of the thread-per-row kernel (run under gpurun)
timeout 600 python -m pytest tests -m gpu -q -x -k "spmv or edge" > gpurun_out/rows_pytest.log 2>&1; tail -1 gpurun_out/rows_pytest.log
for v in 1 2 4 0; do PSC_SPMV_ROWS=$v timeout 300 python bench.py --config 1 --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/rows_$v.json 2>&1; python -c "
import json; d=json.loads(open('gpurun_out/rows_$v.json').read().strip().splitlines()[-1]); print('rows=$v', d['parity'], 'kernel us', round(d['roofline']['kernel_ms']*1e3,2), 'frac', round(d['roofline']['frac'],3), 'step us', round(d['ms_per_step']*1e3,2))"; done
