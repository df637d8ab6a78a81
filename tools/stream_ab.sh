# streaming (lane-per-row) solve on config 4 (run under gpurun)
timeout 900 python -m pytest tests -m gpu -q -x -k "sptrsv or trsv or edge or configs" > gpurun_out/st_pytest.log 2>&1; tail -1 gpurun_out/st_pytest.log
b() { timeout 600 python bench.py --config 4 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/st.json 2>&1; python -c "
import json; d=json.loads(open('gpurun_out/st.json').read().strip().splitlines()[-1]); print('$1', d['parity'], 'kernel ms', round(d['roofline']['kernel_ms'],3), 'GF', round(d['value'],2), 'inspector', round(d['inspector_seconds'],2))" || tail -5 gpurun_out/st.json; }
b smartcut
PSC_TRSV_STREAM_CUT=0 b cut32
