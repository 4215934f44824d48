#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout -s KILL 1500 python -m pytest tests -m "gpu and not slow" -q --timeout 600 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
timeout -s KILL 300 python bench.py --steps 10 --warmup 3 > gpurun_out/bench.log 2>&1
rm -f gpurun_out/bench_apps.log
for w in wator gol gol16k nbody; do timeout -s KILL 300 python bench.py --workload $w --steps 10 --warmup 3 >> gpurun_out/bench_apps.log 2>&1; done
timeout -s KILL 600 python scripts/prof_apps.py gol16k wator > gpurun_out/prof_apps.log 2>&1
