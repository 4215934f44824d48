#!/bin/bash
# A/B of two builds on the microbench phases only:  bash scripts/gpu_ab_lib_mb.sh libA.so [reps]
mkdir -p gpurun_out
rm -f gpurun_out/ab_lib.log
for rep in $(seq 1 ${2:-3}); do
  echo "A $1" >> gpurun_out/ab_lib.log
  DSR_LIBPATH=$1 timeout -s KILL 120 python scripts/prof_mb.py 0 5 0 >> gpurun_out/ab_lib.log 2>&1
  echo "B" >> gpurun_out/ab_lib.log
  timeout -s KILL 120 python scripts/prof_mb.py 0 5 0 >> gpurun_out/ab_lib.log 2>&1
done
