for v in A B C; do
  EDFA_LIB=build_ab/libedfa_$v.so timeout 300 python bench.py --no-cpu-baseline --steps 2 --profile-json gpurun_out/prof_$v.json > gpurun_out/bench_$v.log 2>&1
done
