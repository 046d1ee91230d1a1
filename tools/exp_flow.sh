# A/B of tile-solve kernels / occupancy on the ILU solves (span of one L and U solve)
for v in "EDFA_TILE_KERNEL=pipe" "EDFA_TILE_KERNEL=flow" "EDFA_TILE_KERNEL=flow EDFA_TILE_OCC=1"; do
  echo "== $v" >> gpurun_out/exp_flow.log
  env $v timeout 120 python tools/tiledbg2.py 2>&1 | head -2 >> gpurun_out/exp_flow.log
done
EDFA_TILE_KERNEL=flow timeout 120 python tools/tiledbg3.py > gpurun_out/tiledbg3.log 2>&1
