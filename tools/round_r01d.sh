#!/bin/bash
# round-1d evidence of the current code: bench, ncu launch list, one full capture of the top kernel
mkdir -p gpurun_out
timeout 600 python bench.py > gpurun_out/r01d_bench.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/r01d_bench.log | cut -c1-600
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 9000 --csv \
  --log-file gpurun_out/r01d_ncu_launches.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/r01d_ncu_list.log 2>&1
echo "ncu list rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_tile_flow -s 20 -c 1 \
  -o gpurun_out/r01d_tile_flow_full -f python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/r01d_ncu_full.log 2>&1
echo "ncu full rc=$?"
