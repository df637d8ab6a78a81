# streaming (lane-per-row) solve on config 4 (run under gpurun)
b() { timeout 600 python bench.py --config 4 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/st.json 2>&1; python -c "
import json; d=json.loads(open('gpurun_out/st.json').read().strip().splitlines()[-1]); print('$1', d['parity'], 'kernel ms', round(d['roofline']['kernel_ms'],3), 'GF', round(d['value'],2))" || tail -5 gpurun_out/st.json; }
for k in 8 12 16; do PSC_TRSV_STREAM_K=$k b int1_k$k; done
