#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout -s KILL 1200 python -m pytest tests -m "gpu and not slow" -x -q --timeout 600 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
for f in 4 5 0; do timeout -s KILL 120 python scripts/prof_mb.py $f >> gpurun_out/prof_mb.log 2>&1; done
timeout -s KILL 120 python scripts/prof_mb.py 5 1 >> gpurun_out/prof_mb.log 2>&1
timeout -s KILL 600 ncu --set full --import-source on --clock-control none -k regex:k_mb_new -s 2 -c 1 -o gpurun_out/prof_mbnew python scripts/prof_mb.py 0 > gpurun_out/ncu_mbnew.log 2>&1
timeout -s KILL 600 ncu --set full --import-source on --clock-control none -k regex:k_mb_reduce -s 6 -c 3 -o gpurun_out/prof_reduce python scripts/prof_mb.py 0 > gpurun_out/ncu_reduce.log 2>&1
timeout -s KILL 1200 python -m pytest tests -m "gpu and slow" -x -q --timeout 900 -p no:cacheprovider > gpurun_out/pytest_gpu_slow.log 2>&1
echo "pytest slow exit $?" >> gpurun_out/pytest_gpu_slow.log
