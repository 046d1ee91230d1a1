"""Generate golden artefacts by running the UNMODIFIED reference (hexflow 0.1.0).

Run in the build container only (needs /root/reference):

    python tests/golden/make_golden.py

Writes ``tests/golden/*.npz``.  Each file holds the reference's assembled
blocks plus the stage-1/stage-2 artefacts (restriction sets, G, F, H, the IC
factor of -A_ff, S and its ILU factors), a preconditioner application on a
seeded vector, and the reference Bi-CGStab report.  The inputs are built with
the repo's own seeded generators (``paper_2009_13916_b200.configs``) and then
assembled by the reference's ``assemble``, so the same files also pin the
repo's vectorised assembly.
"""

from __future__ import annotations

import dataclasses
import math
import pathlib
import sys

import numpy as np

HERE = pathlib.Path(__file__).resolve().parent
REPO = HERE.parent.parent
sys.path.insert(0, str(REPO))
sys.path.insert(0, "/root/reference/pkg/src")

import hexflow as hx                                   # noqa: E402
from hexflow.grid import BoundarySpec, _compute_geometry  # noqa: E402
from hexflow.krylov import bicgstab                    # noqa: E402
from hexflow.patterns import base_pattern, static_patterns  # noqa: E402
from hexflow.precond import (BlockLDUPreconditioner, DynamicConfig,  # noqa: E402
                             build_stage1)

from paper_2009_13916_b200 import configs, mesh         # noqa: E402


def put_csr(out, name, M):
    M = M.tocsr()
    out[f"{name}_ptr"] = M.indptr.astype(np.int64)
    out[f"{name}_idx"] = M.indices.astype(np.int64)
    out[f"{name}_val"] = M.data
    out[f"{name}_shape"] = np.array(M.shape, dtype=np.int64)


def put_sets(out, name, sets):
    out[f"{name}_ptr"] = np.concatenate([[0], np.cumsum([s.size for s in sets])]).astype(np.int64)
    out[f"{name}_idx"] = (np.concatenate(sets) if sets else np.empty(0)).astype(np.int64)


def ref_grid(nx, ny, nz, dx, dy, dz, coords=None):
    g = hx.build_structured(nx, ny, nz, dx, dy, dz)
    if coords is not None:
        vol, area = _compute_geometry(coords, g.elem_to_nodes, g.elem_to_faces,
                                      g.face_to_elems, g.face_local)
        g = dataclasses.replace(g, node_coords=coords, elem_volume=vol, face_area=area)
    return g


def record_system(out, s, meta):
    for n in ("A_ff", "A_fc", "A_cf", "A_cc"):
        put_csr(out, n, getattr(s, n))
    out["rhs"] = s.rhs()
    out["free_faces"] = s.free_faces
    out["face_index"] = s.face_index
    out["meta"] = np.array(repr(meta))


def record_precond(out, tag, s, pre, sets):
    put_sets(out, f"{tag}_Q", sets)
    s1, s2 = pre.stage1, pre.stage2
    put_csr(out, f"{tag}_G", s1.G)
    put_csr(out, f"{tag}_F", s1.F)
    put_csr(out, f"{tag}_H", s1.H)
    put_csr(out, f"{tag}_Lff", s1.face_inner.L)
    put_csr(out, f"{tag}_S", s2.S)
    put_csr(out, f"{tag}_LS", s2.schur_inner.L)
    put_csr(out, f"{tag}_US", s2.schur_inner.U)
    out[f"{tag}_shifts"] = np.array([s1.face_inner.pivot_shifts, s2.schur_inner.pivot_shifts])
    out[f"{tag}_density"] = np.array(pre.density)
    rng = np.random.default_rng(77)
    r = rng.standard_normal(s.n_unknowns)
    out[f"{tag}_apply_r"] = r
    out[f"{tag}_apply_y"] = pre.apply(r)
    A = s.full_matrix()
    x, rep = bicgstab(lambda v: A @ v, pre.apply, s.rhs(), tol=1e-8)
    out[f"{tag}_bicg_nit"] = np.array(rep.n_it)
    out[f"{tag}_bicg_x"] = x
    out[f"{tag}_bicg_hist"] = np.array(rep.relres_history)


def case_small_wells():
    """conftest.make_system(4, 4, 2, seed=13, bc_kind="wells"), steady."""
    g = hx.build_structured(4, 4, 2, 1.0, 1.0, 1.0)
    fld = hx.synth_heterogeneous_field(g, 13, (1e-4, 1.0))
    props = hx.FluidRockProps.uniform(g.n_elems, gamma=1.0)
    bc = BoundarySpec(well_columns=[(0, 0, 200.0), (3, 3, 100.0)])
    s = hx.assemble(g, fld, props, bc, dt=math.inf)
    out = {}
    record_system(out, s, dict(kind="small_wells", nx=4, ny=4, nz=2, seed=13))
    out["tensors"] = fld.tensors
    base = base_pattern(s.A_cf)
    variants = {
        "base_fill": dict(patterns=base),                       # reference defaults
        "base_nofill": dict(patterns=base, no_fill=True),
        "dyn14_nofill": dict(dynamic=DynamicConfig(1, 4), no_fill=True),
        "dyn24_nofill": dict(dynamic=DynamicConfig(2, 4), no_fill=True),
        "dyn14_pre": dict(dynamic=DynamicConfig(1, 4), tau_filt=1e-3,
                          filtration="pre", no_fill=True),
        "dyn14_postprod": dict(dynamic=DynamicConfig(1, 4), tau_filt=0.05,
                               filtration="post-product", no_fill=True),
        "dyn14_postschur": dict(dynamic=DynamicConfig(1, 4), tau_filt=0.05,
                                filtration="post-schur", no_fill=True),
        "base_thresh": dict(patterns=base, face_drop_tol=1e-3, schur_drop_tol=1e-3),
    }
    for tag, kw in variants.items():
        pre = BlockLDUPreconditioner.build(s, **kw)
        if "dynamic" in kw:
            sets = dyn_sets(s, kw["dynamic"])
        else:
            sets = kw["patterns"].sets
        record_precond(out, tag, s, pre, sets)
    return out


def dyn_sets(s, cfg):
    A_csc = s.A_ff.tocsc()
    sets = []
    for m in range(s.n_cells):
        lo, hi = s.A_cf.indptr[m], s.A_cf.indptr[m + 1]
        idx, _ = hx.grow_pattern_dynamic(s.A_ff, s.A_cf.indices[lo:hi].astype(np.int64),
                                         s.A_cf.data[lo:hi], cfg, A_csc)
        sets.append(idx)
    return sets


def case_config(idx, n, tags):
    """A scaled-down BASELINE config, assembled by the reference."""
    spec = configs.make(idx, n=n)
    mine = spec.system
    gm = mine.grid
    coords = None if idx != 3 else gm.node_coords
    h = gm.node_coords[1, 0] - gm.node_coords[0, 0] if idx != 3 else 1.0 / n
    g = ref_grid(gm.nx, gm.ny, gm.nz, h, h, h, coords)
    fld = hx.ConductivityField(configs_field(idx, n, gm))
    props = hx.FluidRockProps.uniform(g.n_elems, gamma=1.0)
    bc = BoundarySpec()
    if idx in (1, 2):
        bc.add_plane(g, "x-", pressure=1.0)
        bc.add_plane(g, "x+", pressure=0.0)
    else:
        bc = BoundarySpec(well_columns=[(0, 0, 1.0), (n - 1, n - 1, 0.0)])
    s = hx.assemble(g, fld, props, bc, dt=1.0, p_prev=np.zeros(g.n_elems))
    out = {}
    record_system(out, s, dict(kind=f"config{idx}", n=n))
    out["tensors"] = fld.tensors
    for tag, kw in tags.items():
        if "proto" in kw:
            sets = static_patterns(g, s.face_index, kw["proto"]).sets
            pre = BlockLDUPreconditioner.build(
                s, patterns=hx.PatternSet(sets, "static"), no_fill=True)
        elif "dynamic" in kw:
            pre = BlockLDUPreconditioner.build(s, dynamic=kw["dynamic"], no_fill=True)
            sets = dyn_sets(s, kw["dynamic"])
        else:
            sets = base_pattern(s.A_cf).sets
            pre = BlockLDUPreconditioner.build(s, patterns=base_pattern(s.A_cf), no_fill=True)
        record_precond(out, tag, s, pre, sets)
    return out


def configs_field(idx, n, gm):
    if idx == 1:
        return mesh.Conductivity.homogeneous(gm.n_elems, 1.0).tensors
    if idx == 2:
        return configs.lognormal_aniso_field(gm.n_elems, configs.SEEDS[2]).tensors
    return configs.rotated_tensor_field(gm.n_elems, configs.SEEDS[3] + 1).tensors


def case_static_protos():
    """All five prototypes on a 5x5x5 grid with x-end Dirichlet planes."""
    g = hx.build_structured(5, 5, 5, 1.0, 1.0, 1.0)
    s = hx.assemble(g, hx.ConductivityField.homogeneous(g.n_elems, 1.0),
                    hx.FluidRockProps.uniform(g.n_elems, gamma=1.0),
                    BoundarySpec().add_plane(g, "x-", pressure=2.0).add_plane(
                        g, "x+", pressure=1.0), dt=math.inf)
    out = {}
    record_system(out, s, dict(kind="protos", n=5))
    for p in "ABCDE":
        put_sets(out, f"proto{p}", static_patterns(g, s.face_index, p).sets)
    return out


def main():
    cases = {
        "small_wells": case_small_wells(),
        "config1_n6": case_config(1, 6, {"base": {}}),
        "config2_n8": case_config(2, 8, {"staticA": {"proto": "A"},
                                          "staticB": {"proto": "B"},
                                          "dyn14": {"dynamic": DynamicConfig(1, 4)}}),
        "config3_n5": case_config(3, 5, {"dyn14": {"dynamic": DynamicConfig(1, 4)},
                                          "staticC": {"proto": "C"}}),
        "protos": case_static_protos(),
    }
    for name, out in cases.items():
        np.savez_compressed(HERE / f"{name}.npz", **out)
        print(name, sum(v.nbytes for v in out.values()) // 1024, "KiB raw")


if __name__ == "__main__":
    main()
