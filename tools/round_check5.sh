#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x --timeout 600 -p no:cacheprovider > gpurun_out/pytest_gpu5.log 2>&1
echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu5.log
timeout 400 python bench.py --config 3 --n 48 --steps 1 --warmup 2 --no-cpu-baseline --profile-json gpurun_out/c3_48_prof_r.json > gpurun_out/c3_48_r.log 2>&1
echo "c3 n48 rc=$?"; tail -1 gpurun_out/c3_48_r.log | cut -c1-300
timeout 600 python - > gpurun_out/c4_mid.log 2>&1 <<'PY'
import sys, time
sys.path.insert(0, '.')
import numpy as np, torch
from paper_2009_13916_b200 import configs
import paper_2009_13916_b200 as E
for dims in ((20, 73, 28), (30, 110, 42)):
    case = configs.config4(*dims); s = case.system
    t = time.time()
    ds = E.DeviceSystem.from_host(s)
    pre = E.BlockLDUPreconditioner.build(ds, dynamic=E.DynamicConfig(1, 4), face_drop_tol=1e-3, schur_drop_tol=1e-3)
    x, rep = E.gmres(E.system_operator(ds), pre, s.rhs(), tol=1e-8, restart=50, max_it=2000)
    torch.cuda.synchronize()
    print(dims, "its", rep.n_it, rep.converged, rep.final_relres, "t", time.time() - t, flush=True)
PY
echo "c4 mid rc=$?"; cat gpurun_out/c4_mid.log | tail -3
timeout 1500 python bench.py --config 3 --steps 1 --warmup 1 --no-cpu-baseline --profile-json gpurun_out/c3_full_prof.json > gpurun_out/c3_full.log 2>&1
echo "c3 full rc=$?"; tail -1 gpurun_out/c3_full.log | cut -c1-900
