# full ncu capture of the config-4 streaming solve (run under gpurun, after a plain run)
timeout 600 python bench.py --config 4 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_plain4.json 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:sptrsv_stream -s 2 -c 1 \
  -o gpurun_out/stream_c4 -f python bench.py --config 4 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_c4.log 2>&1
tail -2 gpurun_out/ncu_c4.log
