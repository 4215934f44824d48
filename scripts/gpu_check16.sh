#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout -s KILL 900 python -m pytest tests/test_gpu_inheritance.py tests/test_gpu_apps.py -q -x --timeout 600 -p no:cacheprovider -k "inherit or subtype or subtree or shards" > gpurun_out/pytest_gpu.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
ABL_ONLY=wator-noshift timeout -s KILL 600 python scripts/ablation.py gpurun_out/ablation_noshift.jsonl > gpurun_out/ablation2.log 2>&1
