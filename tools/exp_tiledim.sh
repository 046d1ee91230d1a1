#!/bin/bash
mkdir -p gpurun_out
for td in 8,8,8 8,8,4 16,8,4 8,4,8 4,8,8 16,4,4; do
  EDFA_TILE_DIM=$td timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/td_$td.log 2>&1
  tail -1 gpurun_out/td_$td.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$td', round(d['value'],3), round(d['roofline']['ms_per_launch']*1e3,1), 'us/launch', d['roofline']['kernel'], d['config']['gmres_iterations'])" 2>&1 | tail -1
done
