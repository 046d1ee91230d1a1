#!/bin/bash
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x --timeout 600 -p no:cacheprovider > gpurun_out/pytest_gpu7.log 2>&1
echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu7.log
timeout 600 python bench.py --config 4 --n 24 --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/c4_seq24.log 2>&1
echo "c4 seq rc=$?"; tail -1 gpurun_out/c4_seq24.log | cut -c1-1200
timeout 400 python bench.py --config 3 --n 48 --steps 1 --warmup 2 --no-cpu-baseline --profile-json gpurun_out/c3_48_prof7.json > gpurun_out/c3_48_7.log 2>&1
echo "c3 rc=$?"; tail -1 gpurun_out/c3_48_7.log | cut -c1-300
