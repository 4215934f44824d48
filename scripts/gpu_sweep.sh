#!/bin/bash
# Tuning sweep over prebuilt variants (scripts/sweep_build.py): bash scripts/gpu_sweep.sh "c4 c16 m6"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
rm -f gpurun_out/sweep.log
for rep in 1 2; do
  for v in default $1; do
    lib=""; [ "$v" != default ] && lib=paper_1810_11765_b200/_build/libdsr_$v.so
    echo "variant $v" >> gpurun_out/sweep.log
    DSR_LIBPATH=$lib timeout -s KILL 120 python scripts/prof_mb.py 0 5 1 >> gpurun_out/sweep.log 2>&1
  done
done
for v in default $1; do
  lib=""; [ "$v" != default ] && lib=paper_1810_11765_b200/_build/libdsr_$v.so
  echo "variant $v" >> gpurun_out/sweep.log
  DSR_LIBPATH=$lib timeout -s KILL 300 python scripts/ab_apps.py 0 >> gpurun_out/sweep.log 2>&1
done
