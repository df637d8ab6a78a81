# host vs GPU inspector on every config at full size (run under gpurun)
nproc
for c in 1 2 3 4 5; do timeout 900 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/i$c.json 2>&1; python -c "
import json; d=json.loads(open('gpurun_out/i$c.json').read().strip().splitlines()[-1]); print('config $c', 'host s', round(d['inspector_seconds'],3), 'device s', round(d['inspector_device_seconds'],3), 'equal', d['inspector_device_plan_equal'], 'kernel ms', round(d['roofline']['kernel_ms'],4))" || tail -3 gpurun_out/i$c.json; done
