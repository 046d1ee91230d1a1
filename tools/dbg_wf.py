"""Debug: repeat the wf / tile apply on config 5 (n=20) with blocking launches and report where it fails."""
import os, sys
os.environ.setdefault("CUDA_LAUNCH_BLOCKING", "1")
sys.path.insert(0, ".")
import numpy as np
import paper_2009_13916_b200 as edfa
from paper_2009_13916_b200 import configs
from paper_2009_13916_b200.device import option

n = int(sys.argv[1]) if len(sys.argv) > 1 else 20
case = configs.make(5, n=n)
s = case.system
ds = edfa.DeviceSystem.from_host(s)
pats = edfa.patterns_for(ds, "static", "A")
r = np.random.default_rng(17).standard_normal(s.n_unknowns)
for rep in range(6):
    for wf in (0, 1):
        step = "build"
        try:
            with option("ilu_wf", wf):
                pre = edfa.BlockLDUPreconditioner.build(ds, patterns=pats, no_fill=True)
                step = "apply1"
                y = pre.apply(r)
                step = "apply2"
                y2 = pre.apply(r)
                step = "inner"
                yc = pre.stage2.schur_inner.apply(r[s.n_free_faces:])
            print(f"rep {rep} wf={wf}: ok  |y|={np.linalg.norm(y):.6e} same={np.array_equal(y, y2)}", flush=True)
        except Exception as e:
            print(f"rep {rep} wf={wf}: FAILED at {step}: {e}", flush=True)
            sys.exit(1)
