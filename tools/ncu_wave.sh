# full ncu capture of the config-2 wavefront solve kernel (run under gpurun; after a plain run has passed)
mkdir -p gpurun_out
timeout 300 python bench.py --config 2 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_plain.json 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sptrsv_wave -s 2 -c 1 \
  -o gpurun_out/wave -f python bench.py --config 2 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_wave.log 2>&1
tail -3 gpurun_out/ncu_wave.log
