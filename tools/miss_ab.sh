# config 2: record kernel re-reading only missing operands (PSC_REC_MISSING build flag; run under gpurun)
b() { timeout 300 python bench.py --steps 100 --warmup 5 --no-cpu-baseline > gpurun_out/m.json 2>&1; python -c "
import json; d=json.loads(open('gpurun_out/m.json').read().strip().splitlines()[-1]); print('$1', d['parity'], 'kernel ms', round(d['roofline']['kernel_ms'],4), 'e2e', round(d['e2e']['ms_per_step'],4))"; }
timeout 600 python -m pytest tests -m gpu -q -x -k "sptrsv or trsv or edge or division or bound" 2>&1 | tail -1
b missing1; b missing1_again
cd paper_2111_12243_b200/csrc; touch cuda/kernels.cu; make -s NVEXTRA="-DPSC_REC_MISSING=0" > /dev/null 2>&1; cd ../..
b missing0
cd paper_2111_12243_b200/csrc; touch cuda/kernels.cu; make -s > /dev/null 2>&1
