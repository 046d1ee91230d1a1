#!/bin/bash
# GPU tests + short evidence runs of the newest rows (assembly, threshold factors, config 3/4)
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x --timeout 600 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?"; tail -15 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/smoke.log
EDFA_PHASE_TIMING=1 timeout 400 python bench.py --config 3 --n 48 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/c3_48.log 2>&1
echo "c3 n48 rc=$?"; tail -1 gpurun_out/c3_48.log | cut -c1-700
timeout 600 python bench.py --config 4 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/c4.log 2>&1
echo "c4 rc=$?"; tail -1 gpurun_out/c4.log | cut -c1-900
