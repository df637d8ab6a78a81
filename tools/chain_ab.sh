# single-lane chain: per-row cost of each record loop (run under gpurun)
for v in 0 1; do echo "REC2=$v"; PSC_TRSV_REC2=$v timeout 120 python tools/trsv_chain.py 8192 5; done
