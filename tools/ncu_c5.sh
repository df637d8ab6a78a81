# ncu DRAM bytes of every kernel of one column-split SpMV on config 5 (run under gpurun, after a plain run)
timeout 900 python bench.py --config 5 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_plain5.json 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:spmv_split -s 12 -c 6 --csv \
  python bench.py --config 5 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_c5.csv 2>&1
