#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
rm -f gpurun_out/ab_fpr.log
for rep in 1 2; do
for v in default fpr; do
  lib=""; [ "$v" != default ] && lib=paper_1810_11765_b200/_build/libdsr_$v.so
  echo "variant $v" >> gpurun_out/ab_fpr.log
  DSR_LIBPATH=$lib timeout -s KILL 200 python scripts/ablation.py --one mb '{"name":"bulk","flags":0,"r":5,"reserve":false,"bulk":true}' >> gpurun_out/ab_fpr.log 2>&1
done
done
