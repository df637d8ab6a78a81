# full ncu capture of the config-2 record solve kernel (run under gpurun; after a plain run has passed)
timeout 300 python bench.py --config 2 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_plain.json 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:sptrsv_rec -s 2 -c 1 \
  -o gpurun_out/trsv -f python bench.py --config 2 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_trsv.log 2>&1
tail -3 gpurun_out/ncu_trsv.log
