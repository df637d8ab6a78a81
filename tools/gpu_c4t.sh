#!/bin/bash
mkdir -p gpurun_out
for d in 1 0; do
  echo "== PSC_TRSV_DENSE=$d"
  PSC_TRSV_DENSE=$d timeout 900 python tools/trace_c4.py 1.0 2>&1 | tee gpurun_out/c4_trace_dense$d.log | tail -16
done
