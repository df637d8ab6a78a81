timeout 300 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for T in ${THREADS:-256 512}; do for L in ${LATS:-400 700 1200}; do echo "T=$T LAT=$L"; PSC_TRSV_LAT=$L PSC_TRSV_THREADS=$T timeout 200 python tools/trace_sptrsv.py 2 1.0 2>&1 | sed -n 3,5p; done; done
