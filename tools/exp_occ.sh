#!/bin/bash
# A/B of the dots / IC-pair occupancy knobs on the headline bench (value, dots2 and ic-pair shares)
mkdir -p gpurun_out
for lib in ${LIBS:-base D1 D2 D3 P2 base}; do
  if [ $lib = base ]; then unset EDFA_LIB; else export EDFA_LIB=build_ab/libedfa_$lib.so; fi
  timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/occ_$lib.log 2>&1
  tail -1 gpurun_out/occ_$lib.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; s=r['step_share_of_kernel_time']; k=r['kernel_ms_per_step']; print('$lib', round(d['value'],3), 'dots2 ms', round(s['gs_dots2']*k,2), 'icpair ms', round(s['trsv_ic_pair']*k,2), 'axpy2 ms', round(s['gs_axpy2']*k,2), d['config']['gmres_iterations'])" 2>&1 | tail -1
done
