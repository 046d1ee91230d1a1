#!/bin/bash
# round 2 i: memcheck of the smoke path (tile and wavefront-packed ILU solves), GPU suite, config-5 A/B of the wf layout
mkdir -p gpurun_out
TAG=${1:-r02i}
timeout 900 compute-sanitizer --tool memcheck --error-exitcode 9 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_memcheck_smoke.log 2>&1
echo "memcheck smoke rc=$?"; tail -3 gpurun_out/${TAG}_memcheck_smoke.log
EDFA_OPT_ILU_WF=1 timeout 900 compute-sanitizer --tool memcheck --error-exitcode 9 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_memcheck_smoke_wf.log 2>&1
echo "memcheck smoke wf rc=$?"; tail -3 gpurun_out/${TAG}_memcheck_smoke_wf.log
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/${TAG}_pytest_gpu.log 2>&1; echo "pytest gpu rc=$?"; tail -3 gpurun_out/${TAG}_pytest_gpu.log
for wf in 0 -1; do
  EDFA_OPT_ILU_WF=$wf timeout 900 python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-config2 --profile-json gpurun_out/${TAG}_profile_wf$wf.json > gpurun_out/${TAG}_bench_wf$wf.log 2>&1
  echo "bench wf=$wf rc=$?"; tail -1 gpurun_out/${TAG}_bench_wf$wf.log | cut -c1-600
done
