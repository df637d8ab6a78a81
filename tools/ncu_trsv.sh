# full ncu capture of the config-2 solve kernel (run under gpurun; after a plain run has passed)
V=${1:-1}
PSC_TRSV_REC2=$V timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_plain.json 2>&1 && \
PSC_TRSV_REC2=$V ncu --set full --clock-control none --import-source on -k regex:sptrsv_rec -s 2 -c 1 \
  -o gpurun_out/trsv_v$V -f python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_trsv.log 2>&1
tail -3 gpurun_out/ncu_trsv.log
