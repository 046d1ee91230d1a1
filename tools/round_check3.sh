#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_threshold.py tests/test_gpu_parity.py -m gpu -q -x --timeout 600 -p no:cacheprovider > gpurun_out/pytest_gpu3.log 2>&1
echo "pytest rc=$?"; tail -4 gpurun_out/pytest_gpu3.log
timeout 400 python bench.py --config 3 --n 48 --steps 1 --warmup 2 --no-cpu-baseline --profile-json gpurun_out/c3_48_prof.json > gpurun_out/c3_48c.log 2>&1
echo "c3 rc=$?"; tail -1 gpurun_out/c3_48c.log | cut -c1-600
EDFA_PHASE_TIMING=1 timeout 1200 python bench.py --config 4 --steps 1 --warmup 1 --no-cpu-baseline --single-system --profile-json gpurun_out/c4_prof.json > gpurun_out/c4.log 2>&1
echo "c4 rc=$?"; tail -1 gpurun_out/c4.log | cut -c1-1500
