#!/bin/bash
# tools/ab_variants.sh TAG NAME...: config-5 step of every build_ab/libedfa_NAME.so ("base" = the regular library),
# reporting the per-step kernel times of the profiled warm-up step
mkdir -p gpurun_out
tag=$1; shift
for v in "$@"; do
  lib=""; [ "$v" != base ] && lib=build_ab/libedfa_$v.so
  EDFA_LIB=$lib timeout 600 python bench.py --steps 1 --warmup 2 --no-cpu-baseline --no-config2 \
     --profile-json gpurun_out/${tag}_$v.json > gpurun_out/${tag}_$v.log 2>&1
  python - <<P
import json
try:
    p=json.load(open("gpurun_out/${tag}_$v.json"))["warmup_step"]
    d=json.loads(open("gpurun_out/${tag}_$v.log").read().strip().splitlines()[-1])
    print("$v", "step", round(d["ms_per_step"],1), {k:round(x["ms"],1) for k,x in p.items() if k.startswith("trsv_il") or k in ("trsv_ic_pair","ilu0_factor","product","setup_rows_static")}, d["clocks"]["sm_mhz"])
except Exception as e:
    print("$v", "failed", e)
P
done
