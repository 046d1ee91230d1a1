#!/bin/bash
# A/B of tile-flow compile-time knobs on the headline bench (value, ILU L-solve ms per launch)
mkdir -p gpurun_out
for lib in ${LIBS:-base W8 W14 S0 S64 LS0}; do
  if [ $lib = base ]; then unset EDFA_LIB; else export EDFA_LIB=build_ab/libedfa_$lib.so; fi
  timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/knob_$lib.log 2>&1
  tail -1 gpurun_out/knob_$lib.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$lib', round(d['value'],3), round(d['roofline']['ms_per_launch']*1e3,1), 'us/launch', d['config']['gmres_iterations'])" 2>&1 | tail -1
done
