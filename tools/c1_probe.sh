# config 1: parity (row kernel) vs fast (flag kernel), then ncu of the row kernel (run under gpurun)
for m in parity fast; do
  timeout 300 python bench.py --config 1 --mode $m --steps 50 --warmup 5 --no-cpu-baseline > /tmp/c1.json 2>/tmp/c1.err
  python -c "
import json; d=json.loads(open('/tmp/c1.json').read().strip().splitlines()[-1]); print('$m', 'ms', round(d['ms_per_step'],5), 'launches/step', d['gpu_launches']/d['steps'])"
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:spmv_row -s 3 -c 1 -o gpurun_out/c1_row -f \
  python bench.py --config 1 --mode parity --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_c1.log 2>&1
ncu -i gpurun_out/c1_row.ncu-rep --page raw --csv > gpurun_out/c1_row_raw.csv 2>/dev/null
ncu -i gpurun_out/c1_row.ncu-rep --page source --csv --print-source sass > gpurun_out/c1_row_source.csv 2>/dev/null
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:spmv -c 20 --csv python bench.py --config 1 --mode fast --steps 3 --warmup 3 --no-cpu-baseline 2>/dev/null | grep -E "spmv|Kernel" | tail -6
