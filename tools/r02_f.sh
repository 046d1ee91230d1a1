#!/bin/bash
# round 2 f: tile-shape A/B at 256^3, small configs, the slab path on one GPU, ncu of the direct tile solve
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_configs.py -q -k "c4 or config5 or config4" > gpurun_out/r02f_pytest_configs.log 2>&1
echo "configs tests rc=$?"; tail -3 gpurun_out/r02f_pytest_configs.log
bash tools/r02_ab_tile.sh
for cfg in 1 2; do
  timeout 600 python bench.py --config $cfg --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r02f_bench_c$cfg.log 2>&1
  echo "config $cfg rc=$? $(tail -1 gpurun_out/r02f_bench_c$cfg.log | cut -c1-300)"
done
timeout 900 python bench.py --config 2 --slabs 2 --steps 3 --warmup 2 > gpurun_out/r02f_slabs2.log 2>&1
echo "slabs2 rc=$? $(tail -1 gpurun_out/r02f_slabs2.log | cut -c1-400)"
timeout 900 python bench.py --config 5 --slabs 2 --scaling weak --n 96 --steps 2 --warmup 2 > gpurun_out/r02f_slabs2w.log 2>&1
echo "slabs2 weak rc=$? $(tail -1 gpurun_out/r02f_slabs2w.log | cut -c1-400)"
bash tools/r02_ncu.sh r02f "k_tile_flow" 5
