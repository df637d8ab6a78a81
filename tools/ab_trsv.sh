# A/B of the SpTRSV record loops on config 2 (run under gpurun)
timeout 600 python -m pytest tests -m gpu -q -x -k "sptrsv or trsv or edge" > gpurun_out/ab_pytest.log 2>&1; tail -2 gpurun_out/ab_pytest.log
for v in 0 1; do echo "REC2=$v"; PSC_TRSV_REC2=$v timeout 120 python tools/trsv_chain.py 8192 5; done
for v in 0 1; do PSC_TRSV_REC2=$v timeout 300 python bench.py --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/ab_rec2_$v.json 2>&1; python -c "
import json; d=json.loads(open('gpurun_out/ab_rec2_$v.json').read().strip().splitlines()[-1]); print('rec2=$v', d['parity'], 'kernel ms', round(d['roofline']['kernel_ms'],4), 'e2e ms', round(d['e2e']['ms_per_step'],4))"; done
