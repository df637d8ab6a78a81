# SpTRSV record loop on config 2 (run under gpurun)
timeout 600 python -m pytest tests -m gpu -q -x -k "sptrsv or trsv or edge or division or bound" > gpurun_out/ab_pytest.log 2>&1; tail -1 gpurun_out/ab_pytest.log
timeout 120 python tools/trsv_chain.py 8192 5
for i in 1 2; do timeout 300 python bench.py --steps 100 --warmup 5 --no-cpu-baseline > gpurun_out/ab.json 2>&1; python -c "
import json; d=json.loads(open('gpurun_out/ab.json').read().strip().splitlines()[-1]); print(d['parity'], 'kernel ms', round(d['roofline']['kernel_ms'],4), 'step', round(d['ms_per_step'],4), 'e2e ms', round(d['e2e']['ms_per_step'],4))"; done
