"""Which phase stalls, and does it follow memory-pool growth?"""
import sys, time, json
sys.path.insert(0, "/root/repo")
import torch
from cuda.bindings import runtime as rt
from paper_2009_13916_b200 import configs
from paper_2009_13916_b200.device import DeviceSystem, system_operator
from paper_2009_13916_b200.krylov import gmres
from paper_2009_13916_b200.precond import BlockLDUPreconditioner, patterns_for

case = configs.config2(n=64)
s = case.system
ds = DeviceSystem.from_host(s)
b = torch.from_numpy(s.rhs()).cuda()
_, pool = rt.cudaDeviceGetDefaultMemPool(0)


def reserved():
    e, v = rt.cudaMemPoolGetAttribute(pool, rt.cudaMemPoolAttr.cudaMemPoolAttrReservedMemCurrent)
    return int(v) >> 20


pre = BlockLDUPreconditioner.build(ds, patterns=patterns_for(ds, "static", "A"), no_fill=True)
for it in range(20):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    x, rep = gmres(system_operator(ds), pre, b, tol=1e-8, restart=50)
    torch.cuda.synchronize(); t1 = time.perf_counter()
    print("gmres", round((t1 - t0) * 1e3, 1), "reservedMB", reserved(), flush=True)
for it in range(20):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    pre = BlockLDUPreconditioner.build(ds, patterns=patterns_for(ds, "static", "A"), no_fill=True)
    torch.cuda.synchronize(); t1 = time.perf_counter()
    print("setup", round((t1 - t0) * 1e3, 1), "reservedMB", reserved(), flush=True)
