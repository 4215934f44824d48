#!/bin/bash
# quick round check: build, selected tests, default bench line
mkdir -p gpurun_out
python -c "from paper_1810_11765_b200 import build; build.build()"
timeout 900 python -m pytest ${TESTS:-tests/test_gpu_debug_fault.py} -q --timeout 600 -p no:cacheprovider > gpurun_out/t_check.log 2>&1
echo "exit $?" >> gpurun_out/t_check.log
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench.log 2> gpurun_out/bench.err
echo "bench exit $?" >> gpurun_out/bench.err
