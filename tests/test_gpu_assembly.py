"""GPU parity of the device assembly through the C ABI.

``assemble_device`` against (a) the reference's own blocks (golden fixtures
made by hexflow's ``assemble``, tests/golden/make_golden.py) and (b) the
repo's host restatement ``assembly.assemble`` on the five BASELINE config
generators at small sizes.  Gates: patterns bit-exact (integer work),
values / rhs within 1e-13 relative to the block's max (the reference's BLAS
dot products, numpy's LU inverse and our Cholesky inverse round differently
in the last bits -- the same tolerance t/test_assembly.py grants the
reference against a dense literal assembly), free numbering exact.
"""

from __future__ import annotations

import math

import numpy as np
import pytest
import torch

from conftest import g_blocks, golden, same_csr
from paper_2009_13916_b200 import assembly, configs, mesh

pytestmark = pytest.mark.gpu

TOL = 1e-13


@pytest.fixture(scope="module")
def dev(cuda):
    from paper_2009_13916_b200 import device_assembly
    return device_assembly


def close_csr(M, R, tol=TOL):
    assert same_csr(M, R)
    scale = max(np.abs(R.data).max(), 1e-300) if R.nnz else 1.0
    assert np.abs(M.data - R.data).max(initial=0.0) <= tol * scale


def vec_close(a, b, tol=TOL):
    a = a.cpu().numpy() if isinstance(a, torch.Tensor) else np.asarray(a)
    b = np.asarray(b)
    assert a.shape == b.shape
    assert np.abs(a - b).max(initial=0.0) <= tol * max(np.abs(b).max(initial=0.0), 1.0)


def host_inputs(idx, **kw):
    """Grid / field / props / bc / step of a config generator (configs.py)."""
    if idx == 1:
        n = kw.get("n", 6)
        g = mesh.box_grid(n, n, n, 1.0 / n, 1.0 / n, 1.0 / n)
        return g, mesh.Conductivity.homogeneous(g.n_elems, 1.0), mesh.RockProps(gamma=1.0), \
            mesh.Boundaries(pressure_planes={"x-": 1.0, "x+": 0.0}), 1.0, np.zeros(g.n_elems)
    if idx == 2:
        n = kw.get("n", 8)
        h = 1000.0 / n
        g = mesh.box_grid(n, n, n, h, h, h)
        return g, configs.lognormal_aniso_field(g.n_elems, configs.SEEDS[2]), mesh.RockProps(gamma=1.0), \
            mesh.Boundaries(pressure_planes={"x-": 1.0, "x+": 0.0}), 1.0, np.zeros(g.n_elems)
    if idx == 3:
        n = kw.get("n", 5)
        g = mesh.perturb_interior(mesh.box_grid(n, n, n, 1.0 / n, 1.0 / n, 1.0 / n), 0.2, configs.SEEDS[3])
        return g, configs.rotated_tensor_field(g.n_elems, configs.SEEDS[3] + 1), mesh.RockProps(gamma=1.0), \
            mesh.Boundaries(wells=[(0, 0, 1.0), (n - 1, n - 1, 0.0)]), 1.0, np.zeros(g.n_elems)
    if idx == 4:
        nx, ny, nz = kw.get("dims", (6, 10, 5))
        g = mesh.box_grid(nx, ny, nz, 6.1, 3.05, 0.61)
        bc = mesh.Boundaries(wells=[(0, 0, 200.0), (nx - 1, 0, 200.0), (0, ny - 1, 200.0),
                                    (nx - 1, ny - 1, 200.0), (nx // 2, ny // 2, 100.0)])
        return g, configs.channelised_field(nx, ny, nz, configs.SEEDS[4]), mesh.RockProps(gamma=1.0), bc, \
            0.1, np.full(g.n_elems, 140.0)
    raise ValueError(idx)


def compare(ds, hs):
    for name in ("A_ff", "A_fc", "A_cf", "A_cc"):
        close_csr(getattr(ds, name).to_scipy(), getattr(hs, name))
    close_csr(ds.A_cc_steady.to_scipy(), hs.A_cc_steady)
    assert np.array_equal(ds.face_index.cpu().numpy(), hs.face_index)
    vec_close(ds.rhs(), hs.rhs())
    vec_close(ds.rhs_c_base, hs.rhs_c_base)
    vec_close(ds.accumulation, hs.accumulation)


@pytest.mark.parametrize("fname,idx,n", [("config1_n6", 1, 6), ("config2_n8", 2, 8), ("config3_n5", 3, 5)])
def test_device_assembly_matches_reference_golden(dev, fname, idx, n):
    d = golden(fname)
    g, fld, props, bc, dt, p0 = host_inputs(idx, n=n)
    ds = dev.assemble_device(g, fld, props, bc, dt, p0)
    for name, R in zip(("A_ff", "A_fc", "A_cf", "A_cc"), g_blocks(d)):
        close_csr(getattr(ds, name).to_scipy(), R)
    assert np.array_equal(ds.face_index.cpu().numpy(), d["face_index"])
    vec_close(ds.rhs(), d["rhs"])


@pytest.mark.parametrize("idx,kw", [(1, {"n": 7}), (2, {"n": 12}), (3, {"n": 7}), (4, {"dims": (6, 10, 5)}),
                                    (2, {"n": 20})])
def test_device_assembly_matches_host(dev, idx, kw):
    g, fld, props, bc, dt, p0 = host_inputs(idx, **kw)
    hs = assembly.assemble(g, fld, props, bc, dt, p0)
    ds = dev.assemble_device(g, fld, props, bc, dt, p0, element_ops=True)
    compare(ds, hs)
    n = g.n_elems
    Bi = ds.binv.cpu().numpy().reshape(36, n).T.reshape(n, 6, 6)
    assert np.abs(Bi - hs.ops.Binv).max() <= TOL * np.abs(hs.ops.Binv).max()
    vec_close(ds.elem_volume, g.elem_volume)


def test_steady_and_transient_refresh(dev):
    g, fld, props, bc, _, _ = host_inputs(4, dims=(5, 7, 4))
    hs = assembly.assemble(g, fld, props, bc, math.inf)
    ds = dev.assemble_device(g, fld, props, bc, math.inf)
    compare(ds, hs)
    rng = np.random.default_rng(5)
    for dt in (0.1, 0.37, math.inf, 2.5):
        p = rng.uniform(100, 200, g.n_elems)
        h2 = assembly.update_accumulation(hs, dt, p)
        d2 = dev.update_accumulation_device(ds, dt, p)
        compare(d2, h2)
        assert d2.A_ff is ds.A_ff and d2.A_cf is ds.A_cf      # face blocks shared by identity


def test_flux_planes_and_source(dev):
    g = mesh.box_grid(5, 4, 3, 0.2, 0.25, 1 / 3)
    fld = configs.lognormal_aniso_field(g.n_elems, 7)
    bc = mesh.Boundaries(pressure_planes={"x-": 2.0}, flux_planes={"z+": -0.3, "y-": 0.05})
    props = mesh.RockProps()
    hs = assembly.assemble(g, fld, props, bc, 0.5, np.ones(g.n_elems))
    ds = dev.assemble_device(g, fld, props, bc, 0.5, np.ones(g.n_elems))
    compare(ds, hs)
    # a cell source enters rhs_c as volume * source (hx/assembly.py:279-280)
    src = np.random.default_rng(1).standard_normal(g.n_elems)
    d2 = dev.assemble_device(g, fld, props, bc, math.inf, source=src)
    h2 = assembly.assemble(g, fld, props, bc, math.inf)
    vec_close(d2.rhs_c, h2.rhs_c + g.elem_volume * src)


def test_solve_on_device_assembled_system(dev):
    from paper_2009_13916_b200.device import DeviceSystem, system_operator
    from paper_2009_13916_b200.krylov import gmres
    from paper_2009_13916_b200.precond import BlockLDUPreconditioner, patterns_for
    g, fld, props, bc, dt, p0 = host_inputs(2, n=12)
    hs = assembly.assemble(g, fld, props, bc, dt, p0)
    d = dev.assemble_device(g, fld, props, bc, dt, p0)
    its = []
    for s in (DeviceSystem.from_host(hs), d.system):
        pre = BlockLDUPreconditioner.build(s, patterns=patterns_for(s, "static", "A"), no_fill=True)
        x, rep = gmres(system_operator(s), pre, s.rhs(), tol=1e-8, restart=50)
        its.append(rep.n_it)
        x = x.cpu().numpy() if isinstance(x, torch.Tensor) else x
        b = hs.rhs()
        assert np.linalg.norm(b - hs.full_matrix() @ x) <= 1e-8 * np.linalg.norm(b)
    assert abs(its[0] - its[1]) <= 1


def test_errors(dev):
    g = mesh.box_grid(3, 3, 3, 1.0, 1.0, 1.0)
    fld = mesh.Conductivity.homogeneous(g.n_elems, 1.0)
    with pytest.raises(ValueError):
        dev.assemble_device(g, fld, mesh.RockProps(), mesh.Boundaries(), math.inf)   # singular steady problem
    with pytest.raises(ValueError):
        dev.assemble_device(g, fld, mesh.RockProps(), mesh.Boundaries(pressure_planes={"x-": 1.0}), 0.0)
    c = g.node_coords.copy()
    c[g.elem_to_nodes[13, 6]] = c[g.elem_to_nodes[13, 0]] - 0.5       # invert the centre cell
    bad = mesh.HexGrid(g.nx, g.ny, g.nz, c, g.elem_to_nodes, g.elem_to_faces, g.face_to_elems, g.face_local,
                       g.face_area, g.elem_volume)
    with pytest.raises(ValueError, match="non-positive Jacobian"):
        dev.assemble_device(bad, fld, mesh.RockProps(), mesh.Boundaries(pressure_planes={"x-": 1.0}), math.inf)


@pytest.mark.parametrize("name", ["config2_n6", "config3_n5"])
def test_device_fluxes_and_cfl_match_reference(dev, name):
    """recover_face_fluxes / cfl on the device against the reference's outputs
    (tests/golden/flux_*.npz, made by the unmodified reference) and the
    pinned oracle."""
    from conftest import golden as _golden
    from oracle import edfa_oracle as O
    d = _golden("flux_" + name)
    if name == "config2_n6":
        g, fld, props, bc, _, _ = host_inputs(2, n=6)
    else:
        g, fld, props, bc, _, _ = host_inputs(3, n=5)
    dt = float(d["dt"])
    ds = dev.assemble_device(g, fld, props, bc, dt, d["p_prev"])
    q = dev.recover_face_fluxes_device(ds, d["x"])
    vec_close(q, d["q"], 1e-12)
    nf = ds.n_free_faces
    p_new = torch.from_numpy(d["x"][nf:]).cuda()
    p_old = torch.from_numpy(np.ascontiguousarray(d["p_prev"])).cuda()
    chi, chi_max, dp_max = dev.cfl_device(ds, q, dt, p_new, p_old)
    chi_ref = O.cfl(g.elem_to_faces, g.face_to_elems, d["q"], g.elem_volume, 0.2, dt)
    vec_close(chi, chi_ref, 1e-12)
    assert chi_max == pytest.approx(float(chi_ref.max()), rel=1e-12)
    assert dp_max == float(d["dp_max"])


def test_device_transient_loop_matches_oracle(dev):
    """hx/driver.py run_transient on the device (assembly, refresh, GMRES,
    fluxes, CFL, pressure-change step control) against the same loop driven
    by the oracle on the host."""
    from oracle import edfa_oracle as O
    g, fld, props, bc, _, _ = host_inputs(4, dims=(6, 10, 5))
    kw = dict(p_init=140.0, dt0=0.1, dt_max=5.0, dt_mult=1.1, dp_target=5.0, n_step=4)
    steps, _ = dev.run_transient_device(g, fld, props, bc, precond=dict(pattern="static", prototype="A",
                                                                        no_fill=True), **kw)
    p = np.full(g.n_elems, 140.0)
    dt = 0.1
    base = assembly.assemble(g, fld, props, bc, dt, p)
    o1 = O.build_stage1(base.A_ff, base.A_fc, base.A_cf, sets=O.static_sets(g, base.face_index, "A"),
                        no_fill=True)
    for st in steps:
        s = assembly.update_accumulation(base, dt, p)
        o2 = O.build_stage2(s.A_cc, o1, no_fill=True)
        A, b = s.full_matrix(), s.rhs()
        x, r = O.gmres(lambda v: A @ v, lambda v: O.apply(o1, o2, s.A_fc, s.A_cf, v), b, tol=1e-8, restart=50)
        # dt follows dp_max of solutions that agree to the solver tolerance, not bitwise
        assert st["dt"] == pytest.approx(dt, rel=1e-5)
        assert abs(st["n_it"] - r.n_it) <= 2 and st["converged"]
        pi, pn = s.split(x)
        pif = O.face_pressures(g.n_faces, s.free_faces, s.dirichlet_faces, s.dirichlet_values, pi)
        q = O.recover_face_fluxes(g.elem_to_faces, g.face_to_elems, g.face_local, s.ops.Binv, s.ops.row_sums,
                                  s.ops.diag, pif, pn)
        chi = O.cfl(g.elem_to_faces, g.face_to_elems, q, g.elem_volume, 0.2, dt)
        assert st["cfl_max"] == pytest.approx(float(chi.max()), rel=1e-5)
        dp = float(np.abs(pn - p).max())
        assert st["dp_max"] == pytest.approx(dp, rel=1e-5)
        dt = O.next_dt(dt, 5.0, 1.1, 5.0, dp)
        p = pn
