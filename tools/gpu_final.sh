# round-2 end state (second pass) on the GPU box: tests, smoke, default bench line, reference arm, every config,
# launch list of the default bench, full captures of the config-1 run kernel and the config-4 streaming kernel
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench_default.jsonl 2> gpurun_out/bench_default.err; echo "rc=$?" >> gpurun_out/bench_default.err
timeout 900 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/bench_ref.jsonl 2> gpurun_out/bench_ref.err; echo "rc=$?" >> gpurun_out/bench_ref.err
for c in 1 2 3 4; do timeout 400 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c$c.jsonl 2> gpurun_out/bench_c$c.err; done
timeout 600 python bench.py --config 5 --mode parity --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c5p.jsonl 2> gpurun_out/bench_c5p.err
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file gpurun_out/launches_default.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > /dev/null 2>&1
B="python bench.py --steps 5 --warmup 3 --no-cpu-baseline"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:spmv_run -s 3 -c 1 -o gpurun_out/c1_spmv_run -f $B --config 1 > gpurun_out/ncu_c1.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sptrsv_stream -s 3 -c 1 -o gpurun_out/c4_sptrsv_stream -f $B --config 4 > gpurun_out/ncu_c4.log 2>&1
tail -2 gpurun_out/pytest_gpu.log; tail -1 gpurun_out/smoke.log; cat gpurun_out/bench_c1.jsonl | head -c 600
