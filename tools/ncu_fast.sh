#!/bin/bash
# ncu --set full of the fast-mode merge kernel: tools/ncu_fast.sh CONFIG VARIANT_SPEC [KERNEL_REGEX]
C=${1:-5}
V=${2:-fast:}
K=${3:-spmv_merge}
CMD="python tools/fast_probe.py --config $C --reps 1 --variants $V"
$CMD > gpurun_out/ncu_fast_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:$K -c 3 -o gpurun_out/fast_c$C -f $CMD > gpurun_out/ncu_fast.log 2>&1
echo ncu_rc=$?
