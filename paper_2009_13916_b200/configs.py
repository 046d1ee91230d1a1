"""Seeded synthetic stand-ins for BASELINE.json's five configurations.

The paper measured on a subset of SPE10, which is not in this container;
the BASELINE configs are self-contained synthetic problems.
Every array is generated from ``numpy.random.default_rng(seed)`` with the
seeds below, and fed identically to the CPU oracle and to the GPU path.

Unit convention: permeabilities are passed normalised by
1e-13 m^2 (geometric mean 1), with gamma = 1 and the reference's default
alpha, beta, phi; "one backward-Euler step" uses dt = 1 and p_prev = 0.

Mapping of the restriction techniques:
  config 1 -> base pattern          (Q = column pattern of A_cf^T)
  config 2 -> static prototype "A"  (first technique, the config default)
  config 3 -> dynamic (n_add=2, n_ent=16) (second technique; the CLI's
              (1, 4) budget stagnates at 128^3)
  config 5 inherits config 2's static "A".
Inner solves: IC(0)/ILU(0) (``no_fill=True``, drop tol 0; D5), except config 4,
which runs the reference CLI defaults (dynamic (1, 4), IC(tau)/ILU(tau) with
fill, tau = 1e-3): static A with IC(0)/ILU(0) does not converge on it.
"""

from __future__ import annotations

import math
import time
from dataclasses import dataclass, field

import numpy as np

from . import assembly, mesh

SEEDS = {1: 1001, 2: 1002, 3: 1003, 4: 1004, 5: 1002}


@dataclass
class CaseSpec:
    name: str
    system: object
    precond: dict
    rtol: float = 1e-8
    restart: int = 50
    max_it: int = 2000
    meta: dict = field(default_factory=dict)


HOST_ASSEMBLY = True   # False: configs carry only their inputs (system=None); see inputs_only()


def _assemble(g, fld, props, bc, dt, p_prev):
    """Host assembly plus the inputs it was built from (kept so the device
    assembly, device_assembly.assemble_device, can rebuild the same system)."""
    if not HOST_ASSEMBLY:
        return None, dict(inputs=(g, fld, props, bc, dt, p_prev), host_assembly_s=None)
    t = time.perf_counter()
    s = assembly.assemble(g, fld, props, bc, dt=dt, p_prev=p_prev)
    return s, dict(inputs=(g, fld, props, bc, dt, p_prev), host_assembly_s=time.perf_counter() - t)


def inputs_only(idx: int, **kw) -> CaseSpec:
    """The config's grid, field, properties and boundary conditions without the
    host assembly (``case.system`` is None): large grids are assembled on the
    device (device_assembly.assemble_device(*case.meta["inputs"]))."""
    global HOST_ASSEMBLY
    HOST_ASSEMBLY = False
    try:
        return make(idx, **kw)
    finally:
        HOST_ASSEMBLY = True


def _inner():
    return dict(face_drop_tol=0.0, schur_drop_tol=0.0, no_fill=True)


def lognormal_aniso_field(n_cells, seed, sigma=2.0, kv_kh=0.1):
    rng = np.random.default_rng(seed)
    k = np.exp(rng.normal(0.0, sigma, size=n_cells))
    return mesh.Conductivity.diagonal(k, k, kv_kh * k)


def rotated_tensor_field(n_cells, seed, sigma=1.5):
    """K = R diag(lambda) R^T, lambda_i = exp(N(0, sigma)), R a seeded proper
    rotation (QR of a Gaussian matrix, signs fixed so det R = +1)."""
    rng = np.random.default_rng(seed)
    lam = np.exp(rng.normal(0.0, sigma, size=(n_cells, 3)))
    Q, R = np.linalg.qr(rng.standard_normal((n_cells, 3, 3)))
    Q = Q * np.sign(np.diagonal(R, axis1=1, axis2=2))[:, None, :]
    flip = np.linalg.det(Q) < 0
    Q[flip, :, 0] *= -1.0
    K = np.einsum("nab,nb,ncb->nac", Q, lam, Q)
    return mesh.Conductivity(0.5 * (K + K.transpose(0, 2, 1)))


def config1(n=16):
    g = mesh.box_grid(n, n, n, 1.0 / n, 1.0 / n, 1.0 / n)
    fld = mesh.Conductivity.homogeneous(g.n_elems, 1.0)
    bc = mesh.Boundaries(pressure_planes={"x-": 1.0, "x+": 0.0})
    s, meta = _assemble(g, fld, mesh.RockProps(gamma=1.0), bc, 1.0, np.zeros(g.n_elems))
    return CaseSpec(f"config1-{n}^3-base", s, dict(pattern="base", **_inner()), meta=meta)


def config2(n=64, seed=SEEDS[2], length=1000.0, nz=None):
    """``nz`` > n stacks cubes along z (the weak-scaling grids of BASELINE
    config 5: 64^3 per GPU grown along z so slabs stay z-slabs)."""
    h = length / n
    g = mesh.box_grid(n, n, nz or n, h, h, h)
    fld = lognormal_aniso_field(g.n_elems, seed)
    bc = mesh.Boundaries(pressure_planes={"x-": 1.0, "x+": 0.0})
    s, meta = _assemble(g, fld, mesh.RockProps(gamma=1.0), bc, 1.0, np.zeros(g.n_elems))
    return CaseSpec(f"config2-{n}^3-staticA" if not nz or nz == n else f"config2-{n}x{n}x{nz}-staticA", s,
                    dict(pattern="static", prototype="A", **_inner()), meta=meta)


def config3(n=128, seed=SEEDS[3]):
    """Distorted grid, rotated full-tensor K, injector/producer columns;
    the second (dynamic) restriction technique.  The CLI's dynamic (1, 4)
    budget stagnates at 128^3 (GMRES(50) relres 7.7e-7 after 2000 iterations,
    tools/converge_sweep.py); a larger entry budget of the
    same technique, DynamicConfig(n_add=2, n_ent=16) (hx/precond.py:38-67),
    reaches rtol 1e-8 in ~1000 iterations with IC(0)/ILU(0)."""
    g = mesh.box_grid(n, n, n, 1.0 / n, 1.0 / n, 1.0 / n)
    g = mesh.perturb_interior(g, 0.2, seed)
    fld = rotated_tensor_field(g.n_elems, seed + 1)
    bc = mesh.Boundaries(wells=[(0, 0, 1.0), (n - 1, n - 1, 0.0)])
    s, meta = _assemble(g, fld, mesh.RockProps(gamma=1.0), bc, 1.0, np.zeros(g.n_elems))
    return CaseSpec(f"config3-{n}^3-dynamic2x16", s,
                    dict(pattern="dynamic", n_add=2, n_ent=16, **_inner()), meta=meta)


def channelised_field(nx, ny, nz, seed, sigma=2.5, kv_kh=0.1, n_channel_layers=None, layer_sd=1.5):
    """Layered log-normal background plus high-K sinuous channels in the top
    layers (k x 1e3 inside y0 + a sin(2 pi x / lambda + phi) bands)."""
    rng = np.random.default_rng(seed)
    mu = rng.normal(0.0, layer_sd, size=nz)
    lnk = mu[:, None, None] + rng.normal(0.0, sigma, size=(nz, ny, nx))
    top = n_channel_layers if n_channel_layers is not None else max(1, nz // 2)
    x = np.arange(nx)[None, :]
    y = np.arange(ny)[:, None]
    for k in range(nz - top, nz):
        for _ in range(3):
            y0 = rng.uniform(0, ny)
            a = rng.uniform(0.05, 0.15) * ny
            lam = rng.uniform(0.5, 1.5) * nx
            ph = rng.uniform(0, 2 * np.pi)
            width = rng.uniform(0.02, 0.05) * ny
            band = np.abs(y - (y0 + a * np.sin(2 * np.pi * x / lam + ph))) < width
            lnk[k][band] += np.log(1e3)
    k = np.exp(lnk).ravel()
    return mesh.Conductivity.diagonal(k, k, kv_kh * k)


def config4(nx=60, ny=220, nz=85, seed=SEEDS[4], dt=0.1, sigma=2.5, layer_sd=1.5):
    g = mesh.box_grid(nx, ny, nz, 6.1, 3.05, 0.61)
    fld = channelised_field(nx, ny, nz, seed, sigma=sigma, layer_sd=layer_sd)
    bc = mesh.Boundaries(wells=[(0, 0, 200.0), (nx - 1, 0, 200.0),
                                (0, ny - 1, 200.0), (nx - 1, ny - 1, 200.0),
                                (nx // 2, ny // 2, 100.0)])
    s, meta = _assemble(g, fld, mesh.RockProps(gamma=1.0), bc, dt, np.full(g.n_elems, 140.0))
    # static A with IC(0)/ILU(0) stagnates on this field (z-coupling 10x the
    # x-coupling from the 10:1 cells; the oracle stalls at relres ~1e-4 after
    # 600 iterations on a 12x44x17 box), so config 4 runs the reference CLI's
    # defaults: dynamic (1, 4) patterns, IC(tau)/ILU(tau) with fill, tau = 1e-3
    # (hx/config.py:71-83) -- 37 iterations there
    return CaseSpec(f"config4-{nx}x{ny}x{nz}-dynamic14-transient", s,
                    dict(pattern="dynamic", n_add=1, n_ent=4, face_drop_tol=1e-3, schur_drop_tol=1e-3,
                         no_fill=False),
                    meta=dict(meta, p_init=140.0, n_steps=10, dt0=dt, dt_max=5.0,
                              dt_mult=1.1, dp_target=5.0))


def config5(n=256, seed=SEEDS[5]):
    c = config2(n=n, seed=seed)
    c.name = f"config5-{n}^3-staticA"
    return c


def slab_case(idx: int, n: int, s0: int, s1: int, nz: int | None = None, host: bool = True) -> CaseSpec:
    """The cell layers [s0, s1) of config ``idx``'s n x n x nz grid (default
    nz = n) as a case of their own: same spacing, node coordinates, field
    values (the global seeded draws, sliced) and boundary conditions (x
    planes), so every row whose cells lie inside the slab equals the full
    system's row.  Used by the multi-GPU partition: a rank assembles only its
    extended slab.  Configs 1, 2 and 5 (regular boxes, x-plane Dirichlet)."""
    nz = nz or n
    if idx not in (1, 2, 5):
        raise ValueError("slab_case covers the box configs 1, 2 and 5")
    if not 0 <= s0 < s1 <= nz:
        raise ValueError("slab layers out of range")
    nxy = n * n
    if idx == 1:
        h = 1.0 / n
        g = mesh.box_grid(n, n, s1 - s0, h, h, h, z0_layer=s0)
        fld = mesh.Conductivity.homogeneous(g.n_elems, 1.0)
        precond = dict(pattern="base", **_inner())
    else:
        h = 1000.0 / n
        g = mesh.box_grid(n, n, s1 - s0, h, h, h, z0_layer=s0)
        rng = np.random.default_rng(SEEDS[idx])
        k = np.exp(rng.normal(0.0, 2.0, size=nxy * nz))[s0 * nxy:s1 * nxy]
        fld = mesh.Conductivity.diagonal(k, k, 0.1 * k)
        precond = dict(pattern="static", prototype="A", **_inner())
    bc = mesh.Boundaries(pressure_planes={"x-": 1.0, "x+": 0.0})
    inputs = (g, fld, mesh.RockProps(gamma=1.0), bc, 1.0, np.zeros(g.n_elems))
    s, meta = _assemble(*inputs) if host else (None, dict(inputs=inputs, host_assembly_s=None))
    meta.update(slab=(s0, s1), nz_global=nz)
    return CaseSpec(f"config{idx}-{n}x{n}x{nz}-layers{s0}-{s1}", s, precond, meta=meta)


def make(idx: int, **kw) -> CaseSpec:
    return {1: config1, 2: config2, 3: config3, 4: config4, 5: config5}[idx](**kw)


def steady_equivalent(system):
    return assembly.update_accumulation(system, math.inf)
