"""Per-phase timing of one bench step (patterns / stage 1 / stage 2 / GMRES)."""
import sys, time, json
sys.path.insert(0, '/root/repo')
import torch
from paper_2009_13916_b200 import configs
from paper_2009_13916_b200.device import DeviceSystem, system_operator
from paper_2009_13916_b200.krylov import gmres
from paper_2009_13916_b200.precond import build_stage1, build_stage2, BlockLDUPreconditioner, patterns_for
n = int(sys.argv[1]) if len(sys.argv) > 1 else 64
case = configs.config2(n=n)
s = case.system
ds = DeviceSystem.from_host(s)
b = torch.from_numpy(s.rhs()).cuda()
for it in range(4):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    pats = patterns_for(ds, "static", "A")
    torch.cuda.synchronize(); t1 = time.perf_counter()
    s1 = build_stage1(ds, patterns=pats, no_fill=True)
    torch.cuda.synchronize(); t2 = time.perf_counter()
    pre = BlockLDUPreconditioner(ds, s1, settings=dict(no_fill=True))
    pre.refresh(ds)
    torch.cuda.synchronize(); t3 = time.perf_counter()
    x, rep = gmres(system_operator(ds), pre, b, tol=1e-8, restart=50)
    torch.cuda.synchronize(); t4 = time.perf_counter()
    print(json.dumps(dict(patterns_ms=(t1-t0)*1e3, stage1_ms=(t2-t1)*1e3, stage2_ms=(t3-t2)*1e3, gmres_ms=(t4-t3)*1e3, n_it=rep.n_it)))
