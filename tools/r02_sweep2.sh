#!/bin/bash
# round 2: configs 3/4 at BASELINE size -- Schur-only fill, larger n_ent, the BASELINE-variance config-4 field
mkdir -p gpurun_out
run() { echo "== $*"; timeout 420 python tools/converge_sweep.py "$@" 2>&1 | tail -1 | cut -c1-900; }
{
run --config 3 --n-ent 8 --schur-tol 1e-3 --schur-fill
run --config 3 --n-ent 4 --schur-tol 1e-3 --schur-fill
run --config 3 --n-ent 12
run --config 3 --n-ent 8 --n-add 2
run --config 4 --c4-sigma 1.5811 --c4-layer-sd 0.5
run --config 4 --c4-sigma 1.5811 --c4-layer-sd 0.5 --pattern static --face-tol 0 --schur-tol 0
run --config 4 --c4-sigma 1.5811 --c4-layer-sd 0.5 --face-tol 0 --schur-tol 0
run --config 4 --n-ent 8 --face-tol 1e-3 --schur-tol 1e-3 --schur-fill
} > gpurun_out/r02_sweep2.log 2>&1
