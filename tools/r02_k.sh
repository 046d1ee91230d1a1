#!/bin/bash
mkdir -p gpurun_out
TAG=${1:-r02k}
for n in 20 12 24; do timeout 300 python tools/dbg_wf.py $n > gpurun_out/${TAG}_dbg_wf_$n.log 2>&1; echo "dbg n=$n rc=$?"; tail -3 gpurun_out/${TAG}_dbg_wf_$n.log; done
EDFA_OPT_TILE_DIRECT=2 timeout 900 python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-config2 --profile-json gpurun_out/${TAG}_profile_c5_td2.json > gpurun_out/${TAG}_bench_c5_td2.log 2>&1
echo "bench c5 tile_direct=2 rc=$?"; tail -1 gpurun_out/${TAG}_bench_c5_td2.log | cut -c1-300
