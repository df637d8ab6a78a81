# streaming (lane-per-row) solve on config 4 (run under gpurun)
b() { timeout 600 python bench.py --config 4 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/st.json 2>&1; python -c "
import json; d=json.loads(open('gpurun_out/st.json').read().strip().splitlines()[-1]); print('$1', d['parity'], 'kernel ms', round(d['roofline']['kernel_ms'],3), 'GF', round(d['value'],2))" || tail -5 gpurun_out/st.json; }
b pollall_k8
PSC_TRSV_STREAM_K=12 b pollall_k12
cd paper_2111_12243_b200/csrc; touch cuda/kernels.cu; make -s NVEXTRA="-DPSC_STREAM_POLL1=1" > /dev/null 2>&1; cd ../..
b poll1_k8
cd paper_2111_12243_b200/csrc; touch cuda/kernels.cu; make -s > /dev/null 2>&1
