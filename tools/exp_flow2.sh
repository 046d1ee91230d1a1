for v in A B C; do
  echo "== $v" >> gpurun_out/exp_flow2.log
  EDFA_LIB=build_ab/libedfa_$v.so timeout 120 python tools/tiledbg2.py 2>&1 | head -1 >> gpurun_out/exp_flow2.log
done
EDFA_LIB=build_ab/libedfa_B.so timeout 120 python tools/tiledbg4.py > gpurun_out/tiledbg4.log 2>&1
