# A/B of one config's bench line over environment settings (run under gpurun):
#   bash tools/env_ab.sh CONFIG VAR=VALUE [VAR=VALUE ...]    ("-" = no setting)
C=$1; shift
for v in "$@"; do
  [ "$v" = "-" ] && v=PSC_NONE=1
  env $v timeout 300 python bench.py --config $C --steps 20 --warmup 5 --no-cpu-baseline > /tmp/ab.json 2>/tmp/ab.err
  python -c "
import json; d=json.loads(open('/tmp/ab.json').read().strip().splitlines()[-1]); print('$v', 'ms', round(d['ms_per_step'],4))" || tail -3 /tmp/ab.err
done
