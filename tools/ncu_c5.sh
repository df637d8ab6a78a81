# ncu of the column-split SpMV on config 5 (run under gpurun, after a plain run)
timeout 900 python bench.py --config 5 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_plain5.json 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed,sm__warps_active.avg.pct_of_peak_sustained_active,l1tex__throughput.avg.pct_of_peak_sustained_active --clock-control none -k regex:spmv_split -s 4 -c 4 --csv \
  python bench.py --config 5 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_c5.csv 2>&1
tail -30 gpurun_out/ncu_c5.csv | cut -c1-300
