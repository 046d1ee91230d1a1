for v in "" "EDFA_TILE_NOWAIT=1" "EDFA_TILE_NOWAIT=1 EDFA_TILE_MODE=2" "EDFA_TILE_MODE=1" "EDFA_TILE_OCC=1"; do
  echo "== $v" >> gpurun_out/exp.log
  env $v python tools/tiledbg2.py 2>&1 | head -3 >> gpurun_out/exp.log
done
