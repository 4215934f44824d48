#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
DSR_LIBPATH=paper_1810_11765_b200/_build/libdsr_auw.so timeout -s KILL 600 python -m pytest tests/test_gpu_gol.py -q -x -p no:cacheprovider > gpurun_out/auw_pytest.log 2>&1
rm -f gpurun_out/ab_auw.log
for v in default auw; do
  lib=""; [ "$v" != default ] && lib=paper_1810_11765_b200/_build/libdsr_$v.so
  echo "variant $v" >> gpurun_out/ab_auw.log
  GOL_VARIANTS=handles,tiled_prepare DSR_LIBPATH=$lib timeout -s KILL 300 python scripts/gol_variants.py 3 >> gpurun_out/ab_auw.log 2>&1
done
