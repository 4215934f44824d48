#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout -s KILL 900 python -m pytest tests/test_gpu_gol.py -q -x --timeout 600 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
rm -f gpurun_out/bench_apps.log
for w in gol16k gol16k-bits; do timeout -s KILL 300 python bench.py --workload $w --steps 10 --warmup 3 >> gpurun_out/bench_apps.log 2>&1; done
