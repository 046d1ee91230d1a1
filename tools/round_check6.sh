#!/bin/bash
mkdir -p gpurun_out
timeout 2400 python bench.py --config 5 --steps 1 --warmup 1 --no-cpu-baseline --profile-json gpurun_out/c5_prof.json > gpurun_out/c5.log 2>&1
echo "c5 rc=$?"; tail -1 gpurun_out/c5.log | cut -c1-1200; grep -i "error\|memory" gpurun_out/c5.log | tail -3
