#!/bin/bash
# evidence run of HEAD -- GPU suite, smoke, default bench (config 5), reference arm, other configs,
# ncu launch list and full captures of the hot kernels
mkdir -p gpurun_out
TAG=${1:-r02n}
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/${TAG}_pytest_gpu.log 2>&1; echo "pytest gpu rc=$?"; tail -2 gpurun_out/${TAG}_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/${TAG}_smoke.log
timeout 1500 python bench.py --profile-json gpurun_out/${TAG}_profile.json > gpurun_out/${TAG}_bench.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/${TAG}_bench.log | cut -c1-300
timeout 1200 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/${TAG}_bench_reference.log 2>&1; echo "reference rc=$?"; tail -1 gpurun_out/${TAG}_bench_reference.log | cut -c1-300
for cfg in 1 2; do
  timeout 600 python bench.py --config $cfg --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/${TAG}_bench_c$cfg.log 2>&1
  echo "config $cfg rc=$? $(tail -1 gpurun_out/${TAG}_bench_c$cfg.log | cut -c1-200)"
done
timeout 1500 python bench.py --config 3 --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/${TAG}_bench_c3.log 2>&1
echo "config 3 rc=$? $(tail -1 gpurun_out/${TAG}_bench_c3.log | cut -c1-300)"
timeout 1500 python bench.py --config 4 --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/${TAG}_bench_c4.log 2>&1
echo "config 4 rc=$? $(tail -1 gpurun_out/${TAG}_bench_c4.log | cut -c1-300)"
timeout 1500 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 16000 --csv \
  --log-file gpurun_out/${TAG}_ncu_launches.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-config2 > gpurun_out/${TAG}_ncu_list.log 2>&1
echo "ncu list rc=$?"
bash tools/ncu_kernels.sh $TAG "k_wf k_dots2 k_axpy2 k_spmv_sell k_chain_pair k_product_pf k_setup_rows_reg k_ilu0_sf" 5
