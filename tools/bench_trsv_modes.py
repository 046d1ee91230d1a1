"""Time the inner triangular solves of config 3 (distorted grid, dynamic
patterns) under the solver selections: level-synchronous (EDFA_TRSV_LEVELS),
sync-free thread-per-row / warp-per-row (EDFA_TRSV_WSF forces the sync-free
path).  Usage: python tools/bench_trsv_modes.py N  (run once per env setting)."""
import ctypes as C
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2009_13916_b200 import _lib as L, configs, mesh
from paper_2009_13916_b200.device import ctx, dptr
from paper_2009_13916_b200.device_assembly import assemble_device

n = int(sys.argv[1]) if len(sys.argv) > 1 else 128
g = mesh.perturb_interior(mesh.box_grid(n, n, n, 1 / n, 1 / n, 1 / n), 0.2, configs.SEEDS[3])
fld = configs.rotated_tensor_field(g.n_elems, configs.SEEDS[3] + 1)
bc = mesh.Boundaries(wells=[(0, 0, 1.0), (n - 1, n - 1, 0.0)])
t = time.time()
d = assemble_device(g, fld, mesh.RockProps(gamma=1.0), bc, 1.0, np.zeros(g.n_elems))
torch.cuda.synchronize()
print("assembled", n, "in", round(time.time() - t, 2), "s", flush=True)
lib = L.lib()
f = C.c_void_p()
L.check(lib.edfa_factor_ic(ctx(), d.A_ff.handle, 0.0, 1, C.byref(f)))
nnz, sh, lf, lb = C.c_int64(), C.c_int32(), C.c_int32(), C.c_int32()
L.check(lib.edfa_factor_info(f, C.byref(nnz), C.byref(sh), C.byref(lf), C.byref(lb)))
nf = d.n_free_faces
r = torch.randn(nf, dtype=torch.float64, device="cuda")
y = torch.empty_like(r)
for _ in range(3):
    L.check(lib.edfa_factor_solve(ctx(), f, dptr(r), 1.0, dptr(y)))
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(20):
    L.check(lib.edfa_factor_solve(ctx(), f, dptr(r), 1.0, dptr(y)))
e1.record()
torch.cuda.synchronize()
mode = "levels" if os.environ.get("EDFA_TRSV_LEVELS") else ("wsf" if os.environ.get("EDFA_TRSV_WSF") else "default")
print(f"IC pair solve n={n} rows={nf} levels fwd/bwd={lf.value}/{lb.value} mode={mode}: "
      f"{e0.elapsed_time(e1) / 20:.3f} ms", flush=True)
