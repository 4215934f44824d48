#!/bin/bash
# A/B of two builds of the library on the microbench step and the apps:
#   bash scripts/gpu_ab_lib.sh path/to/libA.so [reps]      (B = the in-tree libdsr.so)
mkdir -p gpurun_out
rm -f gpurun_out/ab_lib.log
for rep in $(seq 1 ${2:-3}); do
  echo "A $1" >> gpurun_out/ab_lib.log
  DSR_LIBPATH=$1 timeout -s KILL 120 python scripts/prof_mb.py 0 5 1 >> gpurun_out/ab_lib.log 2>&1
  echo "B" >> gpurun_out/ab_lib.log
  timeout -s KILL 120 python scripts/prof_mb.py 0 5 1 >> gpurun_out/ab_lib.log 2>&1
done
echo "A apps" >> gpurun_out/ab_lib.log
DSR_LIBPATH=$1 timeout -s KILL 300 python scripts/ab_apps.py 0 >> gpurun_out/ab_lib.log 2>&1
echo "B apps" >> gpurun_out/ab_lib.log
timeout -s KILL 300 python scripts/ab_apps.py 0 >> gpurun_out/ab_lib.log 2>&1
