#!/bin/bash
mkdir -p gpurun_out
TAG=${1:-r02m}
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py -m gpu -x -q > gpurun_out/${TAG}_pytest_gpu.log 2>&1; echo "pytest gpu rc=$?"; tail -3 gpurun_out/${TAG}_pytest_gpu.log
timeout 900 python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-config2 --profile-json gpurun_out/${TAG}_profile_c5_wf.json > gpurun_out/${TAG}_bench_c5_wf.log 2>&1
echo "bench c5 wf rc=$?"; tail -1 gpurun_out/${TAG}_bench_c5_wf.log | cut -c1-400
for n in 128 192; do
  for wf in 0 1; do
    EDFA_OPT_ILU_WF=$wf timeout 600 python bench.py --config 5 --n $n --steps 3 --warmup 2 --no-cpu-baseline --no-config2 --profile-json gpurun_out/${TAG}_profile_c5n${n}_wf$wf.json > gpurun_out/${TAG}_bench_c5n${n}_wf$wf.log 2>&1
    echo "bench c5 n=$n wf=$wf rc=$?"; tail -1 gpurun_out/${TAG}_bench_c5n${n}_wf$wf.log | cut -c1-300
  done
done
