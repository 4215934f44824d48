#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
rm -f gpurun_out/ab_am.log
for v in default am4 am5 am6; do
  lib=""; [ "$v" != default ] && lib=paper_1810_11765_b200/_build/libdsr_$v.so
  echo "variant $v" >> gpurun_out/ab_am.log
  HEAP_GIB=0.5 DSR_LIBPATH=$lib timeout -s KILL 300 python scripts/heap_sweep.py >> gpurun_out/ab_am.log 2>&1
  GOL_VARIANTS=tiled_prepare DSR_LIBPATH=$lib timeout -s KILL 300 python scripts/gol_variants.py 3 >> gpurun_out/ab_am.log 2>&1
done
