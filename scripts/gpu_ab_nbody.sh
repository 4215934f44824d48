#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout -s KILL 600 python -m pytest tests/test_gpu_apps.py tests/test_gpu_static.py -q -x -p no:cacheprovider -k "nbody or Nbody or NBody" > gpurun_out/ab_nb_pytest.log 2>&1
rm -f gpurun_out/ab_nb.log
for rep in 1 2; do
for v in default np1 np4; do
  lib=""; [ "$v" != default ] && lib=paper_1810_11765_b200/_build/libdsr_$v.so
  echo "variant $v" >> gpurun_out/ab_nb.log
  DSR_LIBPATH=$lib timeout -s KILL 200 python scripts/prof_apps.py nbody >> gpurun_out/ab_nb.log 2>&1
done
done
