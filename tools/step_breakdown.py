"""Wall-clock anatomy of one bench step (synchronised sub-phases): system
creation, restriction patterns, stage 1, stage 2, GMRES.

    [EDFA_PHASE_TIMING=1] python tools/step_breakdown.py [config] [n] [reps]

With EDFA_PHASE_TIMING=1 the library also prints its internal phase times
(setup rows, product, IC, Schur, ILU, plans) to stderr.
"""
import json
import pathlib
import sys
import time

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))

import torch  # noqa: E402

from paper_2009_13916_b200 import configs  # noqa: E402
from paper_2009_13916_b200 import device_assembly as DA  # noqa: E402
from paper_2009_13916_b200.device import DeviceSystem, system_operator  # noqa: E402
from paper_2009_13916_b200.krylov import gmres  # noqa: E402
from paper_2009_13916_b200.precond import BlockLDUPreconditioner, build_stage1, patterns_for  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 5
n = int(sys.argv[2]) if len(sys.argv) > 2 else (256 if cfg == 5 else 64)
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
case = configs.inputs_only(cfg, n=n)
dsys = DA.assemble_device(*case.meta["inputs"], element_ops=False)
base = dsys.system
g = case.meta["inputs"][0]
b = base.rhs()


def now():
    torch.cuda.synchronize()
    return time.perf_counter()


for it in range(reps):
    t0 = now()
    ds = DeviceSystem(base.A_ff, base.A_fc, base.A_cf, base.A_cc, rhs=b, topology_src=dsys.topology_inputs)
    ds.set_grid(g.nx, g.ny, g.nz)
    t1 = now()
    pats = patterns_for(ds, "static", "A")
    t2 = now()
    s1 = build_stage1(ds, patterns=pats, no_fill=True)
    t3 = now()
    pre = BlockLDUPreconditioner(ds, s1, settings=dict(no_fill=True))
    pre.refresh(ds)
    t4 = now()
    x, rep = gmres(system_operator(ds), pre, b, tol=1e-8, restart=50)
    t5 = now()
    print(json.dumps(dict(system_ms=(t1 - t0) * 1e3, patterns_ms=(t2 - t1) * 1e3, stage1_ms=(t3 - t2) * 1e3,
                          stage2_ms=(t4 - t3) * 1e3, gmres_ms=(t5 - t4) * 1e3, n_it=rep.n_it)), flush=True)
    del ds, pats, s1, pre, x
