#!/bin/bash
mkdir -p gpurun_out
TAG=${1:-r02l}
for i in 1 2 3 4; do
  CUDA_LAUNCH_BLOCKING=1 timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q > gpurun_out/${TAG}_pytest_blocking_$i.log 2>&1; echo "blocking run $i rc=$?"; grep -n "^E " gpurun_out/${TAG}_pytest_blocking_$i.log | head -5; tail -1 gpurun_out/${TAG}_pytest_blocking_$i.log
done
for i in 1 2 3; do
  timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q > gpurun_out/${TAG}_pytest_async_$i.log 2>&1; echo "async run $i rc=$?"; grep -n "^E " gpurun_out/${TAG}_pytest_async_$i.log | head -5; tail -1 gpurun_out/${TAG}_pytest_async_$i.log
done
