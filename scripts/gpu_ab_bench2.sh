#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout -s KILL 600 python -m pytest tests -q -x -m gpu -k "microbench or reduce or compact" --timeout 300 -p no:cacheprovider > gpurun_out/pytest_sub.log 2>&1
bash scripts/gpu_ab_lib.sh $1 3
timeout -s KILL 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench.log 2>&1
DSR_LIBPATH=$1 timeout -s KILL 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_base.log 2>&1
