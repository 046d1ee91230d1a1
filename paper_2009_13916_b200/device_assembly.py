"""RT0 mixed-hybrid / FV assembly on the device.

``assemble_device`` is hexflow's ``assemble`` (hx/assembly.py:186-311) with
the per-cell work done by libedfa (``edfa_assemble``: element operators,
flux-continuity rows, balance rows, Dirichlet elimination, one thread per
cell / face) and the blocks left in HBM, ready for the EDFA path.  The host
only resolves the boundary specification into per-face codes (the same
``Boundaries.resolve`` the host assembly uses) and uploads the grid arrays.
``update_accumulation_device`` is hx/assembly.py:314-333 on the device.
"""

from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, replace

import numpy as np
import torch

from . import _lib as L
from .device import DeviceCsr, DeviceSystem, ctx, dptr

BC_NONE, BC_PRESSURE, BC_FLUX = 0, 1, 2


@dataclass
class DeviceBlockSystem:
    """Device counterpart of ``BlockSystem`` (hx/assembly.py:135-183): the
    blocks of one step in HBM plus what a time loop needs to refresh it."""

    system: DeviceSystem            # blocks of this step, rhs = [rhs_f; rhs_c]
    A_cc_steady: DeviceCsr
    rhs_f: torch.Tensor
    rhs_c: torch.Tensor
    rhs_c_base: torch.Tensor
    accumulation: torch.Tensor
    elem_volume: torch.Tensor
    face_index: torch.Tensor        # int32, -1 on prescribed-pressure faces
    dirichlet_faces: np.ndarray
    dirichlet_values: np.ndarray
    dt: float
    grid: object
    binv: torch.Tensor | None = None      # [36][n_cells] (SoA)
    row_sums: torch.Tensor | None = None  # [6][n_cells]
    diag: torch.Tensor | None = None      # [6][n_cells]
    dev: dict | None = None               # device grid arrays + per-face boundary values

    @property
    def A_ff(self) -> DeviceCsr:
        return self.system.A_ff

    @property
    def A_fc(self) -> DeviceCsr:
        return self.system.A_fc

    @property
    def A_cf(self) -> DeviceCsr:
        return self.system.A_cf

    @property
    def A_cc(self) -> DeviceCsr:
        return self.system.A_cc

    @property
    def n_free_faces(self) -> int:
        return self.system.n_free_faces

    @property
    def n_cells(self) -> int:
        return self.system.n_cells

    @property
    def n_unknowns(self) -> int:
        return self.system.n_unknowns

    def rhs(self) -> torch.Tensor:
        return self.system.rhs()

    @property
    def topology_inputs(self):
        """(elem_to_faces, face_to_elems, face_index) on the device: what a
        DeviceSystem derives the grid topology from (edfa_grid_topology)."""
        return self.dev["e2f"], self.dev["f2e"], self.face_index

    def to_host(self):
        """The same step as a host ``BlockSystem`` (scipy CSR blocks, numpy
        vectors; element operators not copied) -- what a host application
        holds and hands to the drop-in API."""
        from . import assembly
        n_free = self.n_free_faces
        fidx = self.face_index.cpu().numpy().astype(np.int64)
        free = np.flatnonzero(fidx >= 0)
        assert free.size == n_free
        return assembly.BlockSystem(
            A_ff=self.A_ff.to_scipy(), A_fc=self.A_fc.to_scipy(), A_cf=self.A_cf.to_scipy(),
            A_cc=self.A_cc.to_scipy(), rhs_f=self.rhs_f.cpu().numpy(), rhs_c=self.rhs_c.cpu().numpy(),
            dt=self.dt, free_faces=free, face_index=fidx, dirichlet_faces=self.dirichlet_faces,
            dirichlet_values=self.dirichlet_values, A_cc_steady=self.A_cc_steady.to_scipy(),
            accumulation=self.accumulation.cpu().numpy(), rhs_c_base=self.rhs_c_base.cpu().numpy(),
            ops=None, grid=self.grid)


def _dev(a, dtype) -> torch.Tensor:
    if isinstance(a, torch.Tensor):
        return a.to(device="cuda", dtype=dtype).contiguous()
    a = np.require(np.asarray(a), dtype=np.dtype(str(dtype).split(".")[-1]), requirements=["C", "W"])
    return torch.from_numpy(a).to("cuda", non_blocking=True)


def face_conditions(grid, bc):
    """Per-face boundary codes and values from the boundary specification
    (hx/assembly.py:192-203 checks: prescribed fluxes only on the hull;
    a steady problem needs a prescribed pressure)."""
    dfaces, dvals, nfaces, nvals = bc.resolve(grid)
    n_f = grid.n_faces
    if nfaces.size and np.any(grid.face_to_elems[nfaces, 1] >= 0):
        bad = int(nfaces[np.flatnonzero(grid.face_to_elems[nfaces, 1] >= 0)[0]])
        raise ValueError(f"face {bad} with a prescribed flux is interior")
    code = np.zeros(n_f, np.int8)
    value = np.zeros(n_f)
    code[dfaces] = BC_PRESSURE
    value[dfaces] = dvals
    code[nfaces] = BC_FLUX
    value[nfaces] = nvals
    return code, value, dfaces, dvals


def assemble_device(grid, field, props, bc, dt: float, p_prev=None, source=None,
                    element_ops: bool = True) -> DeviceBlockSystem:
    """Block system for one step (``dt=math.inf``: steady) assembled on the
    device -- hexflow's ``assemble`` (hx/assembly.py:186-311)."""
    if not dt > 0:
        raise ValueError("dt must be positive (math.inf for steady state)")
    code, value, dfaces, dvals = face_conditions(grid, bc)
    if math.isinf(dt) and dfaces.size == 0:
        raise ValueError("steady problem without a prescribed pressure is singular")
    n_e, n_f = grid.n_elems, grid.n_faces
    coords = _dev(grid.node_coords, torch.float64)
    e2n = _dev(grid.elem_to_nodes, torch.int32)
    e2f = _dev(grid.elem_to_faces, torch.int32)
    f2e = _dev(grid.face_to_elems, torch.int32)
    floc = _dev(grid.face_local, torch.int32)
    area = _dev(grid.face_area, torch.float64)
    K = _dev(np.asarray(field.tensors, float).reshape(n_e, 9), torch.float64)
    bc_code = _dev(code, torch.int8)
    bc_val = _dev(value, torch.float64)
    src = None if source is None else _dev(np.broadcast_to(np.asarray(source, float), (n_e,)), torch.float64)
    storage = _dev(np.broadcast_to(np.asarray(props.storage(n_e), float), (n_e,)), torch.float64)

    f64 = dict(dtype=torch.float64, device="cuda")
    fidx = torch.empty(n_f, dtype=torch.int32, device="cuda")
    rhs_f = torch.empty(n_f, **f64)
    rhs_c_base = torch.empty(n_e, **f64)
    vol = torch.empty(n_e, **f64)
    acc = torch.empty(n_e, **f64)
    ops = [torch.empty(k * n_e, **f64) for k in (36, 6, 6)] if element_ops else [None, None, None]

    g = L.HexGridDesc(n_e, n_f, coords.shape[0], dptr(coords), dptr(e2n), dptr(e2f), dptr(f2e), dptr(floc),
                      dptr(area))
    a_in = L.AssemblyIn(dptr(K), float(props.gamma), dptr(bc_code), dptr(bc_val),
                        None if src is None else dptr(src), dptr(storage), 0.0)
    out = L.AssemblyOut(dptr(fidx), dptr(rhs_f), dptr(rhs_c_base), dptr(vol), dptr(acc),
                        *[None if t is None else dptr(t) for t in ops], 0, -1)
    h = [C.c_void_p() for _ in range(4)]
    L.check(L.lib().edfa_assemble(ctx(), C.byref(g), C.byref(a_in), C.byref(out), *[C.byref(x) for x in h]))
    A_ff, A_fc, A_cf, A_cc = (DeviceCsr(x) for x in h)
    n_free = out.n_free
    rhs_f = rhs_f[:n_free]
    ds = DeviceSystem(A_ff, A_fc, A_cf, A_cc, rhs=torch.cat([rhs_f, rhs_c_base]),
                      topology_src=(e2f, f2e, fidx))
    ds.set_grid(grid.nx, grid.ny, grid.nz)
    phi = np.broadcast_to(np.asarray(getattr(props, "porosity", 0.2), float), (n_e,))
    dev = dict(coords=coords, e2n=e2n, e2f=e2f, f2e=f2e, floc=floc, area=area, bc_val=bc_val,
               porosity=_dev(np.ascontiguousarray(phi), torch.float64), n_nodes=coords.shape[0])
    out_sys = DeviceBlockSystem(ds, A_cc, rhs_f, rhs_c_base, rhs_c_base, acc, vol, fidx, dfaces, dvals,
                                math.inf, grid, *ops, dev=dev)
    if math.isinf(dt):
        return out_sys
    return update_accumulation_device(out_sys, dt, p_prev)


def update_accumulation_device(system: DeviceBlockSystem, dt: float, p_prev=None) -> DeviceBlockSystem:
    """New step ``dt``: only A_cc and rhs_c change, the face blocks are shared
    (hx/assembly.py:314-333), so a preconditioner's stage 1 stays valid."""
    if not dt > 0:
        raise ValueError("dt must be positive (math.inf for steady state)")
    n = system.n_cells
    p = None if p_prev is None else _dev(np.broadcast_to(np.asarray(p_prev, float), (n,))
                                         if not isinstance(p_prev, torch.Tensor) else p_prev, torch.float64)
    rhs_c = torch.empty(n, dtype=torch.float64, device="cuda")
    h = C.c_void_p()
    L.check(L.lib().edfa_update_accumulation(ctx(), system.A_cc_steady.handle, dptr(system.accumulation),
                                             dptr(system.rhs_c_base), None if p is None else dptr(p), float(dt),
                                             C.byref(h), dptr(rhs_c)))
    A_cc = DeviceCsr(h)
    old = system.system
    ds = DeviceSystem(old.A_ff, old.A_fc, old.A_cf, A_cc, rhs=torch.cat([system.rhs_f, rhs_c]))
    ds.topology = old.topology
    g = system.grid
    ds.set_grid(g.nx, g.ny, g.nz)
    return replace(system, system=ds, rhs_c=rhs_c, dt=dt)


def _grid_desc(system: DeviceBlockSystem) -> L.HexGridDesc:
    d = system.dev
    return L.HexGridDesc(system.n_cells, system.face_index.numel(), d["n_nodes"],
                         dptr(d["coords"]), dptr(d["e2n"]), dptr(d["e2f"]), dptr(d["f2e"]), dptr(d["floc"]),
                         dptr(d["area"]))


def recover_face_fluxes_device(system: DeviceBlockSystem, x) -> torch.Tensor:
    """Per-face fluxes at the solution x = [pi; p], positive out of the owning
    cell (hx/assembly.py:334-356), on the device."""
    if system.binv is None or system.dev is None:
        raise ValueError("the system was assembled without element operators")
    nf = system.n_free_faces
    x = x if isinstance(x, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(x, dtype=np.float64))
    x = x.to(device="cuda", dtype=torch.float64).contiguous()
    pi, p = x[:nf], x[nf:]
    q = torch.empty(system.face_index.numel(), dtype=torch.float64, device="cuda")
    g = _grid_desc(system)
    L.check(L.lib().edfa_face_fluxes(ctx(), C.byref(g), dptr(system.face_index), dptr(system.dev["bc_val"]),
                                     dptr(system.binv), dptr(system.row_sums), dptr(system.diag), dptr(pi),
                                     dptr(p), dptr(q)))
    return q


def cfl_device(system: DeviceBlockSystem, q: torch.Tensor, dt: float, p_new=None, p_old=None):
    """chi per cell (hx/driver.py:67-71) plus max chi and max |p_new - p_old|."""
    chi = torch.empty(system.n_cells, dtype=torch.float64, device="cuda")
    out = (C.c_double * 2)()
    g = _grid_desc(system)
    L.check(L.lib().edfa_cfl(ctx(), C.byref(g), dptr(q), dptr(system.elem_volume), dptr(system.dev["porosity"]),
                             0.0, float(dt), None if p_new is None else dptr(p_new),
                             None if p_old is None else dptr(p_old), dptr(chi), out))
    return chi, out[0], out[1]


def next_dt(dt: float, dt_max: float, dt_mult: float, dp_target: float, dp_max: float) -> float:
    """TimestepController's rule (hx/driver.py:50-53)."""
    ratio = dt_mult if dp_max <= 0 else min(dt_mult, dp_target / dp_max)
    return min(dt * ratio, dt_max)


def run_transient_device(grid, field, props, bc, *, p_init: float, dt0: float, dt_max: float, dt_mult: float,
                         dp_target: float, n_step: int, precond: dict, tol: float = 1e-8, max_it: int = 2000,
                         restart: int = 50):
    """hx/driver.py:169-230 (``run_transient``) with every array on the device:
    stage 1 once, per step update_accumulation + stage-2 refresh + GMRES, flux
    recovery, CFL and the pressure-change step control.  Returns per-step
    records (dt, iterations, relres, cfl_max, dp_max)."""
    from .device import system_operator
    from .krylov import gmres
    from .precond import BlockLDUPreconditioner, DynamicConfig, patterns_for
    n = grid.n_elems
    p = torch.full((n,), float(p_init), dtype=torch.float64, device="cuda")
    base = assemble_device(grid, field, props, bc, dt0, p)
    opts = dict(precond)
    kind = opts.pop("pattern", "static")
    proto = opts.pop("prototype", "A")
    n_add, n_ent = opts.pop("n_add", 1), opts.pop("n_ent", 4)
    if kind == "dynamic":
        pre = BlockLDUPreconditioner.build(base.system, dynamic=DynamicConfig(n_add, n_ent), **opts)
    else:
        pre = BlockLDUPreconditioner.build(base.system, patterns=patterns_for(base.system, kind, proto), **opts)
    dt, steps = float(dt0), []
    for step in range(n_step):
        s = base if step == 0 else update_accumulation_device(base, dt, p)
        if step:
            pre.refresh(s.system)
        x, rep = gmres(system_operator(s.system), pre, s.rhs(), tol=tol, restart=restart, max_it=max_it)
        nf = s.n_free_faces
        p_new = x[nf:]
        q = recover_face_fluxes_device(s, x)
        _, chi_max, dp_max = cfl_device(s, q, dt, p_new, p)
        steps.append(dict(step=step + 1, dt=dt, n_it=rep.n_it, converged=rep.converged,
                          relres=rep.final_relres, cfl_max=chi_max, dp_max=dp_max))
        dt = next_dt(dt, dt_max, dt_mult, dp_target, dp_max)
        p = p_new
    return steps, x
