#!/bin/bash
# round 2: A/B of the ILU tile-solve shapes on config 5 (256^3)
mkdir -p gpurun_out
for m in 1 2 0; do
  EDFA_OPT_TILE_DIRECT=$m timeout 900 python bench.py --steps 2 --warmup 2 --no-cpu-baseline --no-config2 \
    --profile-json gpurun_out/r02_ab_tile$m.json > gpurun_out/r02_ab_tile$m.log 2>&1
  echo "mode $m rc=$? $(tail -1 gpurun_out/r02_ab_tile$m.log | cut -c1-200)"
done
