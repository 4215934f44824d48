#!/bin/bash
# A/B of variant builds (scripts/sweep_build.py): microbench phases, Wa-Tor heap sweep, GoL variants.
#   bash scripts/gpu_ab_free.sh "fr1 fr2"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout -s KILL 600 python -m pytest tests/test_gpu_gol.py -q -x -p no:cacheprovider > gpurun_out/ab_pytest_gol.log 2>&1
rm -f gpurun_out/ab.log
for v in default $1; do
  lib=""; [ "$v" != default ] && lib=paper_1810_11765_b200/_build/libdsr_$v.so
  echo "variant $v" >> gpurun_out/ab.log
  DSR_LIBPATH=$lib timeout -s KILL 200 python scripts/mb_variants.py 5 bulk >> gpurun_out/ab.log 2>&1
  DSR_LIBPATH=$lib timeout -s KILL 200 python scripts/heap_sweep.py >> gpurun_out/ab.log 2>&1
  DSR_LIBPATH=$lib timeout -s KILL 300 python scripts/gol_variants.py 3 >> gpurun_out/ab.log 2>&1
done
