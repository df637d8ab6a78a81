# config 2: back-off of the solving warp that shares the halo warp's sub-partition (run under gpurun)
b() { timeout 300 python bench.py --steps 100 --warmup 5 --no-cpu-baseline > gpurun_out/w.json 2>&1; python -c "
import json; d=json.loads(open('gpurun_out/w.json').read().strip().splitlines()[-1]); print('$1', d['parity'], 'kernel ms', round(d['roofline']['kernel_ms'],4))"; }
b base
for ns in 32 100 300; do
cd paper_2111_12243_b200/csrc; touch cuda/kernels.cu; make -s NVEXTRA="-DPSC_W3_SLEEP=$ns" > /dev/null 2>&1; cd ../..
b sleep$ns
done
cd paper_2111_12243_b200/csrc; touch cuda/kernels.cu; make -s > /dev/null 2>&1
