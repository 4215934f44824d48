#!/bin/bash
# parity tests against a variant library, then the sweep: bash scripts/gpu_variant_test.sh name
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
DSR_LIBPATH=paper_1810_11765_b200/_build/libdsr_$1.so timeout -s KILL 900 python -m pytest tests -q -x -m gpu --timeout 300 -p no:cacheprovider > gpurun_out/pytest_variant.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_variant.log
bash scripts/gpu_sweep.sh "$1"
