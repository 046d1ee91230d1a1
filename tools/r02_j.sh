#!/bin/bash
# round 2 j: wf layout A/B at config 5 / 2 / 1 with per-kernel profiles, trsv + wf tests
mkdir -p gpurun_out
TAG=${1:-r02j}
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py -m gpu -x -q > gpurun_out/${TAG}_pytest_gpu.log 2>&1; echo "pytest gpu rc=$?"; tail -3 gpurun_out/${TAG}_pytest_gpu.log
EDFA_OPT_ILU_WF=-1 timeout 900 python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-config2 --profile-json gpurun_out/${TAG}_profile_c5_wf.json > gpurun_out/${TAG}_bench_c5_wf.log 2>&1
echo "bench c5 wf rc=$?"; tail -1 gpurun_out/${TAG}_bench_c5_wf.log | cut -c1-400
for cfg in 2 1; do
  for wf in 0 1; do
    EDFA_OPT_ILU_WF=$wf timeout 600 python bench.py --config $cfg --steps 5 --warmup 3 --no-cpu-baseline --profile-json gpurun_out/${TAG}_profile_c${cfg}_wf$wf.json > gpurun_out/${TAG}_bench_c${cfg}_wf$wf.log 2>&1
    echo "bench c$cfg wf=$wf rc=$?"; tail -1 gpurun_out/${TAG}_bench_c${cfg}_wf$wf.log | cut -c1-400
  done
done
