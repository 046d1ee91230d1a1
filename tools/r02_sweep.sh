#!/bin/bash
# round 2: convergence of configs 3/4 at BASELINE size under reference-native options
mkdir -p gpurun_out
run() { echo "== $*"; timeout 420 python tools/converge_sweep.py "$@" 2>&1 | tail -2; }
{
run --config 4 --face-tol 1e-4 --schur-tol 1e-4 --fill
run --config 4 --n-ent 8 --face-tol 1e-3 --schur-tol 1e-3 --fill
run --config 4 --solver bicgstab
run --config 4 --pattern static --face-tol 1e-3 --schur-tol 1e-3 --fill
run --config 3 --solver bicgstab
run --config 3 --n-ent 8
run --config 3 --pattern static
run --config 3 --face-tol 1e-3 --schur-tol 1e-3 --fill
} > gpurun_out/r02_sweep.log 2>&1
