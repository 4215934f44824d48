#!/bin/bash
# allocator-heavy GPU tests, then an A/B of the in-tree library against $1
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout -s KILL 900 python -m pytest tests -q -x -m gpu --timeout 300 -p no:cacheprovider -k "not fulllength" > gpurun_out/pytest_sub.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_sub.log
bash scripts/gpu_ab_lib.sh $1 ${2:-3}
