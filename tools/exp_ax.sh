for v in A B C D; do
  echo "== $v" >> gpurun_out/exp_ax.log
  EDFA_LIB=build_ab/libedfa_$v.so timeout 120 python tools/axdbg.py 2>&1 | head -3 >> gpurun_out/exp_ax.log
done
