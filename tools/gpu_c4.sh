# config-4 solve: GPU tests, bench line (run under gpurun)
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
timeout 400 python bench.py --config 4 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c4.jsonl 2> gpurun_out/bench_c4.err
python -c "
import json; d=json.loads(open('gpurun_out/bench_c4.jsonl').read().strip().splitlines()[-1]); print('c4 ms', round(d['ms_per_step'],3), 'frac', round(d['roofline']['frac'],4))" || tail -3 gpurun_out/bench_c4.err
timeout 500 python tools/trace_c4.py 1.0 2>&1 | tail -4
