#!/bin/bash
mkdir -p gpurun_out
PSC_TRSV_WAVE=a timeout 600 python tools/trace_sptrsv.py 2 1.0 > gpurun_out/wave_trace.log 2>&1; head -3 gpurun_out/wave_trace.log
PSC_TRSV_TRACE_ROWS=0 PSC_TRSV_WAVE=a timeout 600 python tools/trace_sptrsv.py 2 1.0 > gpurun_out/wave_trace0.log 2>&1; head -2 gpurun_out/wave_trace0.log
