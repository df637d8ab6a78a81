# experiment: solve units on 16 lanes per warp (PSC_TRSV_HALF_LANES build) vs 32
b() { PSC_TRSV_REC2=$1 timeout 300 python bench.py --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/h.json 2>&1; python -c "
import json; d=json.loads(open('gpurun_out/h.json').read().strip().splitlines()[-1]); print('$2 rec2=$1', d['parity'], 'kernel ms', round(d['roofline']['kernel_ms'],4))"; }
b 0 full32
cd paper_2111_12243_b200/csrc; touch cuda/kernels.cu; make -s NVEXTRA="-DPSC_TRSV_HALF_LANES=1" > /dev/null 2>&1; cd ../..
PSC_TRSV_THREADS=256 b 0 half16
PSC_TRSV_THREADS=256 b 1 half16
cd paper_2111_12243_b200/csrc; touch cuda/kernels.cu; make -s > /dev/null 2>&1
