#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
rm -f gpurun_out/ab3.log
for rep in 1 2; do
for v in default bfr3; do
  lib=""; [ "$v" != default ] && lib=paper_1810_11765_b200/_build/libdsr_$v.so
  echo "variant $v" >> gpurun_out/ab3.log
  DSR_LIBPATH=$lib timeout -s KILL 200 python scripts/mb_variants.py 5 bulk >> gpurun_out/ab3.log 2>&1
done
done
timeout -s KILL 1800 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=10 > gpurun_out/pytest_gpu.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
