# config-5 fast SpMV: launch list of one bench step, and a full capture of the three flag-kernel passes (run under gpurun)
timeout 300 python bench.py --config 5 --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/c5_plain.jsonl 2>&1 || exit 1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct --clock-control none --csv \
  --log-file gpurun_out/c5_launches.csv python bench.py --config 5 --steps 2 --warmup 1 --no-cpu-baseline > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:spmv_flag -c 3 -o gpurun_out/c5_flag -f \
  python bench.py --config 5 --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_c5.log 2>&1
tail -2 gpurun_out/ncu_c5.log
ncu -i gpurun_out/c5_flag.ncu-rep --page raw --csv > gpurun_out/c5_flag_raw.csv 2>/dev/null
ncu -i gpurun_out/c5_flag.ncu-rep --page source --csv --print-source sass > gpurun_out/c5_flag_source.csv 2>/dev/null
