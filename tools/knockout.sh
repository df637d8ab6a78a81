# latency knock-outs of the converged record loop (chain test; run under gpurun)
cd paper_2111_12243_b200/csrc
for v in "" "-DPSC_X_NODIV" "-DPSC_X_NOSENT" "-DPSC_X_NOACC" "-DPSC_X_NOSTG" "-DPSC_X_NODIV -DPSC_X_NOSENT -DPSC_X_NOACC -DPSC_X_NOSTG"; do
  touch cuda/kernels.cu; make -s NVEXTRA="$v" > /dev/null 2>&1 || echo "build failed $v"
  echo "== $v"; (cd ../.. && PSC_TRSV_REC2=0 timeout 120 python tools/trsv_chain.py 8192 5)
done
touch cuda/kernels.cu; make -s > /dev/null 2>&1
