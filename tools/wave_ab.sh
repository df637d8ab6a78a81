# config-2 wave solve A/B over environment settings (run under gpurun): one line per setting
for v in "$@"; do
  env $v timeout 120 python bench.py --config 2 --steps 20 --warmup 5 --no-cpu-baseline > /tmp/ab.json 2>/tmp/ab.err
  python -c "
import json,sys; d=json.loads(open('/tmp/ab.json').read().strip().splitlines()[-1]); print('$v', 'ms', round(d['ms_per_step'],4))" || tail -3 /tmp/ab.err
done
