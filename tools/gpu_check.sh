# GPU tests + every config's bench line (no CPU baseline) (run under gpurun)
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
for c in ${CONFIGS:-1 2 3 4 5}; do
  timeout 400 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c$c.jsonl 2> gpurun_out/bench_c$c.err
  python -c "
import json; d=json.loads(open('gpurun_out/bench_c$c.jsonl').read().strip().splitlines()[-1]); print('config $c', d['config']['mode'], 'ms', round(d['ms_per_step'],4), 'frac', round(d['roofline']['frac'],3), 'e2e ms', round(d['e2e']['ms_per_step'],3))" || tail -3 gpurun_out/bench_c$c.err
done
