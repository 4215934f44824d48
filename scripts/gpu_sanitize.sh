#!/bin/bash
# compute-sanitizer runs on small configurations of every app (results checked against the oracle)
mkdir -p gpurun_out
python -c "from paper_1810_11765_b200 import build; build.build()"
for tool in memcheck racecheck synccheck initcheck; do
  timeout 1200 compute-sanitizer --tool $tool --print-limit 20 --error-exitcode 9 python scripts/sanitize_small.py > gpurun_out/sanitize_$tool.log 2>&1
  echo "compute-sanitizer --tool $tool exit $?" >> gpurun_out/sanitize_$tool.log
done
