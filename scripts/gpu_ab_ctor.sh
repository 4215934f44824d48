#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
rm -f gpurun_out/ab_ctor.log
for rep in 1 2; do
for v in default rnf; do
  lib=""; [ "$v" != default ] && lib=paper_1810_11765_b200/_build/libdsr_$v.so
  echo "variant $v" >> gpurun_out/ab_ctor.log
  DSR_LIBPATH=$lib timeout -s KILL 200 python scripts/mb_variants.py 5 bulk >> gpurun_out/ab_ctor.log 2>&1
done
done
