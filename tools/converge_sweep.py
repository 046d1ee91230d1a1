#!/usr/bin/env python
"""Convergence of EDFA + GMRES(50) on one BASELINE config under a given set of
reference-native preconditioner options (hx/config.py:71-84): pattern kind,
n_add/n_ent/it_max, face/schur drop tolerance, fill.  Prints one JSON line.

    python tools/converge_sweep.py --config 3 [--n 128] [--pattern dynamic --n-ent 4]
                                   [--drop-tol 1e-3 --fill] [--max-it 2000]
"""
from __future__ import annotations

import argparse
import json
import pathlib
import sys
import time

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, required=True)
    ap.add_argument("--n", type=int, default=None)
    ap.add_argument("--dims", default=None, help="nx,ny,nz (config 4)")
    ap.add_argument("--pattern", default=None)
    ap.add_argument("--prototype", default="A")
    ap.add_argument("--n-add", type=int, default=1)
    ap.add_argument("--n-ent", type=int, default=4)
    ap.add_argument("--it-max", type=int, default=None)
    ap.add_argument("--face-tol", type=float, default=None)
    ap.add_argument("--schur-tol", type=float, default=None)
    ap.add_argument("--fill", action="store_true", help="fill-in for both inner factorisations")
    ap.add_argument("--schur-fill", action="store_true", help="fill-in for the Schur ILU only (face IC no_fill)")
    ap.add_argument("--max-it", type=int, default=2000)
    ap.add_argument("--restart", type=int, default=50)
    ap.add_argument("--solver", default="gmres", choices=["gmres", "bicgstab"])
    ap.add_argument("--c4-sigma", type=float, default=None, help="config 4: std of ln K per cell")
    ap.add_argument("--c4-layer-sd", type=float, default=None, help="config 4: std of the per-layer mean of ln K")
    a = ap.parse_args()

    import torch

    from paper_2009_13916_b200 import configs
    from paper_2009_13916_b200.device import DeviceSystem, system_operator
    from paper_2009_13916_b200.krylov import bicgstab, gmres
    from paper_2009_13916_b200.precond import BlockLDUPreconditioner, DynamicConfig, patterns_for

    t0 = time.perf_counter()
    if a.config == 4:
        kw = {}
        if a.dims:
            nx, ny, nz = (int(v) for v in a.dims.split(","))
            kw = dict(nx=nx, ny=ny, nz=nz)
        if a.c4_sigma is not None:
            kw["sigma"] = a.c4_sigma
        if a.c4_layer_sd is not None:
            kw["layer_sd"] = a.c4_layer_sd
        case = configs.config4(**kw)
    else:
        case = configs.make(a.config, **({"n": a.n} if a.n else {}))
    t_gen = time.perf_counter() - t0
    p = dict(case.precond)
    pattern = a.pattern or p["pattern"]
    ftol = a.face_tol if a.face_tol is not None else p.get("face_drop_tol", 0.0)
    stol = a.schur_tol if a.schur_tol is not None else p.get("schur_drop_tol", 0.0)
    if a.fill or a.schur_fill or a.face_tol is not None or a.schur_tol is not None:
        face_nf, schur_nf = not a.fill, not (a.fill or a.schur_fill)
    else:
        face_nf = schur_nf = p.get("no_fill", True)
    ds = DeviceSystem.from_host(case.system)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    from paper_2009_13916_b200.precond import build_stage1
    if pattern == "dynamic":
        s1 = build_stage1(ds, dynamic=DynamicConfig(a.n_add, a.n_ent, a.it_max), face_drop_tol=ftol, no_fill=face_nf)
    else:
        s1 = build_stage1(ds, patterns=patterns_for(ds, pattern, a.prototype), face_drop_tol=ftol, no_fill=face_nf)
    pre = BlockLDUPreconditioner(ds, s1, settings=dict(tau_filt=0.0, filtration="none", schur_drop_tol=stol,
                                                       no_fill=schur_nf))
    pre.refresh(ds)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    solve = gmres if a.solver == "gmres" else bicgstab
    kw = dict(restart=a.restart) if a.solver == "gmres" else {}
    x, rep = solve(system_operator(ds), pre, ds.rhs(), tol=case.rtol, max_it=a.max_it, **kw)
    torch.cuda.synchronize()
    t3 = time.perf_counter()
    h = rep.relres_history
    print(json.dumps(dict(config=a.config, name=case.name, n_dof=ds.n_unknowns, pattern=pattern,
                          n_add=a.n_add, n_ent=a.n_ent, it_max=a.it_max, face_tol=ftol, schur_tol=stol,
                          face_no_fill=face_nf, schur_no_fill=schur_nf, solver=a.solver, restart=a.restart, its=rep.n_it,
                          converged=rep.converged, relres=rep.final_relres, density=pre.density,
                          t_gen=round(t_gen, 2), t_setup=round(t2 - t1, 3), t_solve=round(t3 - t2, 3),
                          hist_every_100=[h[k] for k in range(0, len(h), 100)])), flush=True)


if __name__ == "__main__":
    main()
