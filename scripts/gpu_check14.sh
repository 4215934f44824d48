#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout -s KILL 900 python -m pytest tests/test_gpu_gol.py -q --timeout 600 -p no:cacheprovider -m "gpu and not slow" > gpurun_out/pytest_gpu.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
rm -f gpurun_out/bench_apps.log
timeout -s KILL 300 python bench.py --workload gol --steps 50 --warmup 3 >> gpurun_out/bench_apps.log 2>&1
