#!/bin/bash
# End-of-round evidence: headline bench (config 2) and the other configs at full size
mkdir -p gpurun_out
timeout 600 python bench.py > gpurun_out/final_c2.log 2>&1; echo "c2 rc=$?"; tail -1 gpurun_out/final_c2.log | cut -c1-700
timeout 300 python bench.py --config 1 --no-cpu-baseline > gpurun_out/final_c1.log 2>&1; echo "c1 rc=$?"; tail -1 gpurun_out/final_c1.log | cut -c1-400
timeout 1500 python bench.py --config 3 --steps 1 --warmup 1 --no-cpu-baseline --profile-json gpurun_out/final_c3_prof.json > gpurun_out/final_c3.log 2>&1; echo "c3 rc=$?"; tail -1 gpurun_out/final_c3.log | cut -c1-900
