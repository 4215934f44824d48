#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout -s KILL 600 python -m pytest tests/test_gpu_allocator.py -q -x -p no:cacheprovider > gpurun_out/ab_leaf_pytest.log 2>&1
rm -f gpurun_out/ab_leaf.log
for rep in 1 2; do
for v in default lanes; do
  lib=""; [ "$v" != default ] && lib=paper_1810_11765_b200/_build/libdsr_$v.so
  echo "variant $v" >> gpurun_out/ab_leaf.log
  DSR_LIBPATH=$lib timeout -s KILL 200 python scripts/ablation.py --one mb '{"name":"bulk","flags":0,"r":5,"reserve":false,"bulk":true}' >> gpurun_out/ab_leaf.log 2>&1
done
done
