bash scripts/gpu_ab.sh "0 128" 2
for f in 0 128; do timeout -s KILL 300 python scripts/ab_apps.py $f >> gpurun_out/ab.log 2>&1; done
