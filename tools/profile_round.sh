# ncu evidence for profiles/ (run under gpurun): the launch list of the default
# bench command, then one full capture of every config's dominant kernel, each
# after the same command line has exited 0 without ncu.
set -u
mkdir -p gpurun_out/prof
B="python bench.py --steps 5 --warmup 3 --no-cpu-baseline"
$B > gpurun_out/prof/plain_c2.json 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/prof/launches_c2.csv $B > gpurun_out/prof/ncu_launch.log 2>&1
cap() {  # config kernel-regex name
  $B --config $1 > gpurun_out/prof/plain_c$1.json 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:$2 -s 3 -c 1 -o gpurun_out/prof/$3 -f $B --config $1 > gpurun_out/prof/ncu_$3.log 2>&1
  echo "c$1 $2 rc=$?"
}
cap 2 sptrsv_rec c2_sptrsv_rec
cap 1 spmv_row c1_spmv_row
cap 3 spmv_group c3_spmv_group
cap 4 sptrsv_stream c4_sptrsv_stream
cap 5 spmv_split_chunk c5_spmv_split_chunk
ls -la gpurun_out/prof
