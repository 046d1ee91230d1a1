#!/bin/bash
# round 2: config 3 pattern budgets / fill, config 4 prototypes at BASELINE size
mkdir -p gpurun_out
run() { echo "== $*"; timeout 600 python tools/converge_sweep.py "$@" 2>&1 | tail -1 | cut -c1-1200; }
{
run --config 3 --n-ent 8
run --config 3 --n-ent 12
run --config 3 --n-ent 8 --n-add 2
run --config 3 --n-ent 16 --n-add 2
run --config 3 --n-ent 8 --face-tol 1e-3 --schur-tol 1e-3 --fill
run --config 4 --n-ent 16 --n-add 4 --face-tol 0 --schur-tol 0
run --config 4 --pattern static --prototype C --face-tol 0 --schur-tol 0
run --config 4 --pattern static --prototype E --face-tol 0 --schur-tol 0
} > gpurun_out/r02_sweep3.log 2>&1
