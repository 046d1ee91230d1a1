#!/bin/bash
# short evidence run of HEAD: GPU suite, smoke, default bench (config 5 + the config-2 leg + CPU baseline),
# ncu launch list and a full capture of the ILU solve kernel
mkdir -p gpurun_out
TAG=${1:-r04h}
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/${TAG}_pytest_gpu.log 2>&1; echo "pytest gpu rc=$?"; tail -2 gpurun_out/${TAG}_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/${TAG}_smoke.log
timeout 1500 python bench.py --profile-json gpurun_out/${TAG}_profile.json > gpurun_out/${TAG}_bench.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/${TAG}_bench.log | cut -c1-300
timeout 1500 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 16000 --csv \
  --log-file gpurun_out/${TAG}_ncu_launches.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-config2 > gpurun_out/${TAG}_ncu_list.log 2>&1
echo "ncu list rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k 'regex:^k_wf_pf$' -s 40 -c 2 \
    -o gpurun_out/${TAG}_k_wf_c5 -f python bench.py --config 5 --steps 1 --warmup 1 --no-cpu-baseline --no-config2 \
    > gpurun_out/${TAG}_k_wf_c5.log 2>&1
echo "ncu k_wf rc=$?"
