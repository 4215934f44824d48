#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout -s KILL 1500 python -m pytest tests -m "gpu and not slow" -q --timeout 600 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
timeout -s KILL 300 python bench.py --steps 10 --warmup 3 > gpurun_out/bench.log 2>&1
timeout -s KILL 600 ncu --set full --clock-control none -k regex:"k_mb_reduce|k_compact" -s 12 -c 6 -o gpurun_out/r01_mb_reduce2 python scripts/prof_targets.py mb > gpurun_out/ncu2.log 2>&1
