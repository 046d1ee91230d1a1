#!/bin/bash
# Round evidence on one B200: ncu launch list + one full capture of the top kernel,
# then bench lines for the other BASELINE configs (evidence runs, not the headline).
set -u
mkdir -p gpurun_out
TAG=${TAG:-r01c}
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 9000 --csv \
  --log-file gpurun_out/${TAG}_ncu_launches.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/${TAG}_ncu_list.log 2>&1
echo "ncu list rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_tile_flow -s 20 -c 1 \
  -o gpurun_out/${TAG}_tile_flow_full -f python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/${TAG}_ncu_full.log 2>&1
echo "ncu full rc=$?"
for c in 1 3 4 5; do
  timeout 1200 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/${TAG}_bench_c$c.log 2>&1
  echo "config $c rc=$?"; tail -1 gpurun_out/${TAG}_bench_c$c.log | cut -c1-400
done
