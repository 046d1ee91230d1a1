#!/bin/bash
mkdir -p gpurun_out
timeout 400 python bench.py --config 3 --n 48 --steps 1 --warmup 2 --no-cpu-baseline --profile-json gpurun_out/c3_48_prof.json > gpurun_out/c3_48b.log 2>&1
echo "c3 rc=$?"; tail -1 gpurun_out/c3_48b.log | cut -c1-400
EDFA_PHASE_TIMING=1 timeout 900 python bench.py --config 4 --steps 1 --warmup 2 --no-cpu-baseline --profile-json gpurun_out/c4_prof.json > gpurun_out/c4.log 2>&1
echo "c4 rc=$?"; tail -1 gpurun_out/c4.log | cut -c1-1500
timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/c2.log 2>&1
echo "c2 rc=$?"; tail -1 gpurun_out/c2.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['e2e']['value'], json.dumps(d.get('assembly')))"
