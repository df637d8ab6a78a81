# full ncu capture of the config-3 SpMV kernel (run under gpurun, after a plain run)
timeout 300 python bench.py --config 3 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_plain3.json 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:spmv_group -s 2 -c 1 \
  -o gpurun_out/spmv_c3g -f python bench.py --config 3 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_c3.log 2>&1
tail -2 gpurun_out/ncu_c3.log
