#!/bin/bash
# Microbench phase times of several library builds, interleaved:
#   bash scripts/gpu_ab_multi.sh tag reps lib1.so lib2.so ...   ("-" = the in-tree build)
T=$1; R=$2; shift 2
mkdir -p gpurun_out
out=gpurun_out/abm_$T.log
rm -f $out
for rep in $(seq 1 $R); do
  for lib in "$@"; do
    echo "LIB $lib" >> $out
    if [ "$lib" = "-" ]; then timeout -s KILL 120 python scripts/prof_mb.py 0 5 0 >> $out 2>&1
    else DSR_LIBPATH=$lib timeout -s KILL 120 python scripts/prof_mb.py 0 5 0 >> $out 2>&1; fi
  done
done
