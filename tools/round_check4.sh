#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x --timeout 600 -p no:cacheprovider > gpurun_out/pytest_gpu4.log 2>&1
echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu4.log
for v in 0 1; do
  if [ $v = 1 ]; then export EDFA_TRSV_WSF=1; fi
  timeout 400 python bench.py --config 3 --n 48 --steps 1 --warmup 2 --no-cpu-baseline --profile-json gpurun_out/c3_48_prof_$v.json > gpurun_out/c3_48_$v.log 2>&1
  echo "c3 wsf=$v rc=$?"; tail -1 gpurun_out/c3_48_$v.log | cut -c1-300
done
