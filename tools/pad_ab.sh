# experiment: halo warp on another SMSP (PSC_HALO_PAD idle warps)
b() { PSC_TRSV_REC2=$1 timeout 300 python bench.py --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/h.json 2>&1; python -c "
import json; d=json.loads(open('gpurun_out/h.json').read().strip().splitlines()[-1]); print('$2 rec2=$1', d['parity'], 'kernel ms', round(d['roofline']['kernel_ms'],4))"; }
b 0 pad0; b 1 pad0
for pad in 1 2 3; do
cd paper_2111_12243_b200/csrc; touch cuda/kernels.cu; make -s NVEXTRA="-DPSC_HALO_PAD=$pad" > /dev/null 2>&1; cd ../..
b 0 pad$pad; b 1 pad$pad
done
cd paper_2111_12243_b200/csrc; touch cuda/kernels.cu; make -s > /dev/null 2>&1
