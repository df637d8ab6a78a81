# experiment: outlined IEEE division in the record loop (PSC_TRSV_OUTLINED build flag)
b() { timeout 300 python bench.py --steps 100 --warmup 5 --no-cpu-baseline > gpurun_out/h.json 2>&1; python -c "
import json; d=json.loads(open('gpurun_out/h.json').read().strip().splitlines()[-1]); print('$1', d['parity'], 'kernel ms', round(d['roofline']['kernel_ms'],4), 'e2e', round(d['e2e']['ms_per_step'],4))"; }
timeout 600 python -m pytest tests -m gpu -q -x -k "sptrsv or trsv or edge or division" > gpurun_out/o_pytest.log 2>&1; tail -1 gpurun_out/o_pytest.log
b outlined1; timeout 120 python tools/trsv_chain.py 8192 5
cd paper_2111_12243_b200/csrc; touch cuda/kernels.cu; make -s NVEXTRA="-DPSC_TRSV_OUTLINED=0" > /dev/null 2>&1; cd ../..
b outlined0; timeout 120 python tools/trsv_chain.py 8192 5
b outlined0_again
cd paper_2111_12243_b200/csrc; touch cuda/kernels.cu; make -s > /dev/null 2>&1; cd ../..
b outlined1_again
