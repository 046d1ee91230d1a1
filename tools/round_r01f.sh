#!/bin/bash
# round-1e: dots at 2 blocks per SM — GPU tests, smoke, bench, ncu launch list
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r01f_pytest_gpu.log 2>&1; echo "pytest gpu rc=$?"; tail -3 gpurun_out/r01f_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r01f_smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/r01f_smoke.log
timeout 600 python bench.py > gpurun_out/r01f_bench.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/r01f_bench.log | cut -c1-900
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 9000 --csv \
  --log-file gpurun_out/r01f_ncu_launches.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/r01f_ncu_list.log 2>&1
echo "ncu list rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_dots2 -s 40 -c 1 \
  -o gpurun_out/r01f_dots2_full -f python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/r01f_ncu_full.log 2>&1
echo "ncu full rc=$?"
