#!/bin/bash
# Full-length BASELINE runs against the oracle (tests/test_gpu_fulllength.py)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
DSR_FULL=1 timeout -s KILL 3000 python -m pytest tests/test_gpu_fulllength.py -v -s --timeout 2400 -p no:cacheprovider --durations=0 > gpurun_out/fulllength.log 2>&1
echo "pytest exit $?" >> gpurun_out/fulllength.log
