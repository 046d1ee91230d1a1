#!/bin/bash
# Convergence of configs 3/4 at BASELINE size under reference-native options (tools/converge_sweep.py);
# the outcome is summarised in profiles/r02_convergence.json.
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
