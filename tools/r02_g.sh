#!/bin/bash
# round 2 g: full GPU suite, smoke, default bench (config 5), launch list, step anatomy, dynamic-setup ncu (config 3)
mkdir -p gpurun_out
TAG=${1:-r02g}
bash tools/r02_check.sh $TAG
EDFA_PHASE_TIMING=1 timeout 600 python tools/step_breakdown.py 5 256 2 > gpurun_out/${TAG}_step_breakdown.log 2>&1
echo "breakdown rc=$?"; tail -4 gpurun_out/${TAG}_step_breakdown.log
timeout 1500 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 16000 --csv \
  --log-file gpurun_out/${TAG}_ncu_launches.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-config2 > gpurun_out/${TAG}_ncu_list.log 2>&1
echo "ncu list rc=$?"
timeout 900 ncu --set full --clock-control none -k regex:k_setup_rows -c 1 -o gpurun_out/${TAG}_setup_rows_dyn_c3 -f \
  python tools/converge_sweep.py --config 3 --max-it 5 > gpurun_out/${TAG}_ncu_dyn.log 2>&1
echo "ncu dyn rc=$?"
