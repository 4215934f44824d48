#!/bin/bash
# A/B of a library build against the in-tree one on the microbench phases and the apps,
# after the allocator / app GPU tests at the in-tree build:
#   bash scripts/gpu_ab_lib_all.sh tag libA.so [reps]
T=$1; A=$2; R=${3:-3}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$T.log 2>&1
timeout -s KILL 1200 python -m pytest tests/test_gpu_allocator.py tests/test_gpu_gol.py tests/test_gpu_apps.py tests/test_gpu_debug_fault.py -q -x -m gpu --timeout 600 -p no:cacheprovider > gpurun_out/pytest_$T.log 2>&1
echo "pytest rc $?" >> gpurun_out/pytest_$T.log
bash scripts/gpu_ab_multi.sh $T $R $A -
out=gpurun_out/aba_$T.log; rm -f $out
for rep in $(seq 1 $R); do
  echo "LIB $A" >> $out; DSR_LIBPATH=$A timeout -s KILL 300 python scripts/ab_apps.py 0 wator >> $out 2>&1
  DSR_LIBPATH=$A timeout -s KILL 300 python scripts/ab_gol.py 3 >> $out 2>&1
  echo "LIB -" >> $out; timeout -s KILL 300 python scripts/ab_apps.py 0 wator >> $out 2>&1
  timeout -s KILL 300 python scripts/ab_gol.py 3 >> $out 2>&1
done
