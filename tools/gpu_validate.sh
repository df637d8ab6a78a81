# full GPU validation: tests, default bench line, reference arm, every config (run under gpurun)
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
timeout 300 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; tail -1 gpurun_out/bench_default.json
timeout 300 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/bench_ref.json 2>&1; tail -1 gpurun_out/bench_ref.json
bash tools/spmv_configs.sh
timeout 400 python bench.py --config 4 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c4.json 2>&1; tail -1 gpurun_out/bench_c4.json
timeout 300 python tools/trace_sptrsv.py 2 > gpurun_out/trace.log 2>&1; head -3 gpurun_out/trace.log
