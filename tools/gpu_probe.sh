# latency primitives + SpTRSV trace (diagnostics; run under gpurun)
nvcc -O3 -gencode arch=compute_100a,code=sm_100a tools/latency_bench.cu -o /tmp/lb && /tmp/lb
timeout 300 python tools/trace_sptrsv.py 2
