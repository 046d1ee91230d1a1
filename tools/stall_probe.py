"""Diagnose step-time outliers: per step, wall time vs summed kernel time."""
import ctypes
import json
import sys
import time

sys.path.insert(0, "/root/repo")
import torch

from paper_2009_13916_b200 import _lib, configs
from paper_2009_13916_b200.device import DeviceSystem, ctx, system_operator
from paper_2009_13916_b200.krylov import gmres
from paper_2009_13916_b200.precond import BlockLDUPreconditioner, patterns_for

lib = _lib.lib()
SLOW = []
if "--wrap" in sys.argv:
    for _name in _lib._SIGS:
        _fn = getattr(lib, _name)

        def _w(*a, _fn=_fn, _name=_name):
            t = time.perf_counter()
            r = _fn(*a)
            dt = time.perf_counter() - t
            if dt > 0.02:
                SLOW.append((_name, round(dt * 1e3, 1)))
            return r
        setattr(lib, _name, _w)
if "--nogc" in sys.argv:
    import gc
    gc.disable()
if "--reserve" in sys.argv:
    big = torch.empty(0)
    from paper_2009_13916_b200.device import ctx as _c
    _c()
    ptr = ctypes.c_void_p()
    rt = ctypes.CDLL("libcudart.so.12") if False else None
case = configs.config2(n=int(sys.argv[1]) if len(sys.argv) > 1 else 64)
s = case.system
ds = DeviceSystem.from_host(s)
b = torch.from_numpy(s.rhs()).cuda()
c = ctx()


def report(reset=1):
    n = lib.edfa_ctx_profile_report(c, None, 0, 0)
    buf = ctypes.create_string_buffer(int(n))
    lib.edfa_ctx_profile_report(c, buf, n, reset)
    return json.loads(buf.value.decode())


lib.edfa_ctx_profile(c, 1)
report()
for it in range(int(sys.argv[2]) if len(sys.argv) > 2 and sys.argv[2].isdigit() else 12):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    cpu0 = time.process_time()
    pats = patterns_for(ds, "static", "A")
    pre = BlockLDUPreconditioner.build(ds, patterns=pats, no_fill=True)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    x, rep = gmres(system_operator(ds), pre, b, tol=1e-8, restart=50)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    cpu1 = time.process_time()
    p = report()
    k = sum(v["ms"] for v in p.values())
    top = sorted(p.items(), key=lambda kv: -kv[1]["ms"])[:int(__import__("os").environ.get("TOPN", "3"))]
    slow, SLOW[:] = list(SLOW), []
    print(json.dumps(dict(slow=slow, setup_ms=round((t1 - t0) * 1e3, 1), gmres_ms=round((t2 - t1) * 1e3, 1),
                          kernel_ms=round(k, 1), cpu_ms=round((cpu1 - cpu0) * 1e3, 1),
                          top={a: round(v["ms"], 1) for a, v in top})), flush=True)
