# config 1: staged (coalesced) vs per-thread loads in the thread-per-row kernel (run under gpurun)
b() { timeout 300 python bench.py --config 1 --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/r.json 2>&1; python -c "
import json; d=json.loads(open('gpurun_out/r.json').read().strip().splitlines()[-1]); print('$1', d['parity'], 'kernel us', round(d['roofline']['kernel_ms']*1e3,2), 'frac', round(d['roofline']['frac'],3))"; }
b base
PSC_SPMV_STAGED=1 b staged
PSC_SPMV_STAGED=1 timeout 600 python -m pytest tests -m gpu -q -x -k "spmv or configs or acceptance or edge" 2>&1 | tail -1
