#!/bin/bash
# full ncu captures of the hot kernels on the config-5 (256^3) step and the setup kernels on config 2
# usage: tools/ncu_kernels.sh TAG "regex1 regex2 ..." [config]
mkdir -p gpurun_out
TAG=$1; KS=$2; CFG=${3:-5}
for k in $KS; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k -s 2 -c 1 \
    -o gpurun_out/${TAG}_${k}_c${CFG} -f python bench.py --config $CFG --steps 1 --warmup 1 --no-cpu-baseline --no-config2 \
    > gpurun_out/${TAG}_${k}_c${CFG}.log 2>&1
  echo "ncu $k rc=$?"
done
