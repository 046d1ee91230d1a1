#!/bin/bash
mkdir -p gpurun_out
for n in 64 128; do
  timeout 300 python tools/bench_trsv_modes.py $n 2>&1 | tail -1
  EDFA_TRSV_LEVELS=1 timeout 300 python tools/bench_trsv_modes.py $n 2>&1 | tail -1
  EDFA_TRSV_WSF=1 timeout 300 python tools/bench_trsv_modes.py $n 2>&1 | tail -1
done
