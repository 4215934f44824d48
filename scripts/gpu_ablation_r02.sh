#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout -s KILL 3000 python scripts/ablation.py gpurun_out/ablation.jsonl > gpurun_out/ablation.log 2>&1
echo "ablation exit $?" >> gpurun_out/ablation.log
