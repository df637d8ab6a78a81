# config 3: per-kernel times of one multiply (run under gpurun, after a plain run)
timeout 600 python bench.py --config 3 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/c3p.json 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:spmv -s 4 -c 4 --csv python bench.py --config 3 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/c3l.csv 2>&1
