# round-2 end state on the GPU box: tests, smoke, default bench line, reference arm, every config, launch list
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
tail -2 gpurun_out/pytest_gpu.log; tail -1 gpurun_out/smoke.log
