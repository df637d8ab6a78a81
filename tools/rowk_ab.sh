# config 1: bulk L2 prefetch in the thread-per-row kernel (run under gpurun)
b() { timeout 300 python bench.py --config 1 --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/r.json 2>&1; python -c "
import json; d=json.loads(open('gpurun_out/r.json').read().strip().splitlines()[-1]); print('$1', d['parity'], 'kernel us', round(d['roofline']['kernel_ms']*1e3,2), 'frac', round(d['roofline']['frac'],3))"; }
b base
cd paper_2111_12243_b200/csrc; touch cuda/kernels.cu; make -s NVEXTRA="-DPSC_ROWK_PF=1" > /dev/null 2>&1; cd ../..
b prefetch
cd paper_2111_12243_b200/csrc; touch cuda/kernels.cu; make -s > /dev/null 2>&1
