#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python bench.py --config 5 --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/f2_c5.log 2>&1; echo "c5 rc=$?"; tail -1 gpurun_out/f2_c5.log | cut -c1-700
timeout 600 python bench.py --slabs 1 --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/f2_s1.log 2>&1; echo "slabs1 rc=$?"; tail -1 gpurun_out/f2_s1.log | cut -c1-500
timeout 600 python bench.py --slabs 2 --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/f2_s2.log 2>&1; echo "slabs2 rc=$?"; tail -1 gpurun_out/f2_s2.log | cut -c1-500
