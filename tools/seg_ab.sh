# SpMV segmented-plan kernels on config 3 (run under gpurun)
timeout 600 python -m pytest tests -m gpu -q -x -k "spmv or edge" > gpurun_out/seg_pytest.log 2>&1; tail -2 gpurun_out/seg_pytest.log
for v in 2 3; do PSC_SPMV_SEGLANE=$v timeout 300 python bench.py --config 3 --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/seg_$v.json 2>&1; python -c "
import json; d=json.loads(open('gpurun_out/seg_$v.json').read().strip().splitlines()[-1]); print('seg=$v', d['parity'], 'kernel ms', round(d['roofline']['kernel_ms'],4), 'frac', round(d['roofline']['frac'],3))"; done
for c in 1 5; do timeout 300 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/c$c.json 2>&1; python -c "
import json; d=json.loads(open('gpurun_out/c$c.json').read().strip().splitlines()[-1]); print('config $c', d['parity'], 'kernel ms', round(d['roofline']['kernel_ms'],4), 'frac', round(d['roofline']['frac'],3))"; done
