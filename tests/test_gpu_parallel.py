"""Slab-partitioned EDFA + GMRES on the GPU (parallel.CudaSlab through libedfa).

Several slabs are held by one process on one device (their halo copies are
local; no kernel waits on another launch), which exercises exactly the
per-rank device work of a multi-GPU run.  The reference is the oracle's
EDFA with slab-block-diagonal inner factors.
"""

from __future__ import annotations

import numpy as np
import pytest
import scipy.sparse as sp

from oracle import edfa_oracle as O
from slab_cpu import block_jacobi_reference

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def par(cuda):
    from paper_2009_13916_b200 import _lib, parallel
    _lib.lib()
    return parallel


def _system(n=6, which=2):
    from paper_2009_13916_b200 import configs
    return configs.make(which, n=n).system


def _solve(par, s, parts, kind="static", proto="A", dynamic=None):
    from paper_2009_13916_b200.precond import DynamicConfig
    dyn = DynamicConfig(*dynamic[:2]) if dynamic else None
    lays = par.build_layouts(s, parts, halo=par.halo_layers(kind, proto, dyn))
    solver = par.SlabSolver(lays, par.LocalComm(parts), kind=kind, prototype=proto, dynamic=dyn)
    solver.build()
    xs, rep = solver.solve(tol=1e-8, restart=50)
    x = par.scatter_solution(lays, xs, s.n_free_faces, s.n_cells)
    return lays, solver, x, rep


def _sets(s, kind, proto):
    if kind == "base":
        return O.base_sets(s.A_cf)
    return O.static_sets(s.grid, s.face_index, proto)


@pytest.mark.parametrize("parts", [1, 2, 3])
def test_slabs_match_block_jacobi_oracle(par, parts):
    s = _system(6)
    lays, solver, x, rep = _solve(par, s, parts)
    sets = _sets(s, "static", "A")
    x_ref, rep_ref, S_bj = block_jacobi_reference(s, lays, sets)
    assert rep.converged and rep_ref.converged
    assert abs(rep.n_it - rep_ref.n_it) <= 2, (rep.n_it, rep_ref.n_it)
    A = s.full_matrix()
    assert np.linalg.norm(s.rhs() - A @ x) <= 1e-8 * np.linalg.norm(s.rhs()) * 1.0001
    assert np.linalg.norm(x - x_ref) <= 1e-7 * np.linalg.norm(x_ref)
    # block-Jacobi Schur blocks: the slab's S~[own, own] from its extended stage 1
    for lay, part in zip(lays, solver.parts):
        mine = part.S_own.to_scipy()
        ref = S_bj.tocsr()[lay.own_cells][:, lay.own_cells]
        d = abs(mine - ref)
        assert d.max() <= 1e-12 * abs(ref).max()


def test_one_slab_equals_fused_solver(par):
    import paper_2009_13916_b200 as E
    s = _system(8)
    _, _, x1, rep1 = _solve(par, s, 1)
    ds = E.DeviceSystem.from_host(s)
    pre = E.BlockLDUPreconditioner.build(ds, patterns=E.patterns_for(ds, "static", "A"), no_fill=True)
    x2, rep2 = E.gmres(E.system_operator(ds), pre, s.rhs(), tol=1e-8, restart=50)
    assert abs(rep1.n_it - rep2.n_it) <= 1
    assert np.linalg.norm(x1 - x2) <= 1e-9 * np.linalg.norm(x2)


@pytest.mark.parametrize("kind,proto", [("base", "A"), ("static", "B")])
def test_slabs_other_patterns(par, kind, proto):
    s = _system(6, which=1 if kind == "base" else 2)
    lays, _, x, rep = _solve(par, s, 2, kind=kind, proto=proto)
    x_ref, rep_ref, _ = block_jacobi_reference(s, lays, _sets(s, kind, proto))
    assert abs(rep.n_it - rep_ref.n_it) <= 2
    assert np.linalg.norm(x - x_ref) <= 1e-7 * np.linalg.norm(x_ref)


def test_slabs_dynamic(par):
    s = _system(5, which=3)
    lays, _, x, rep = _solve(par, s, 2, kind="dynamic", dynamic=(1, 4))
    x_ref, rep_ref, _ = block_jacobi_reference(s, lays, dynamic=(1, 4, None))
    assert abs(rep.n_it - rep_ref.n_it) <= 2
    assert np.linalg.norm(x - x_ref) <= 1e-7 * np.linalg.norm(x_ref)


def test_slab_static_pattern_on_extended_box(par):
    """The device static-pattern kernel on the extended box yields the global
    sets of the slab's own cells (ext numbering)."""
    from paper_2009_13916_b200.patterns import static_patterns_device
    s = _system(8)
    lays = par.build_layouts(s, 3, halo=par.halo_layers("static", "A"))
    glob = _sets(s, "static", "A")
    for lay in lays:
        part = par.CudaSlab(lay)
        sets = static_patterns_device(part.ext.topology, "A").sets
        for c_ext in lay.blocks["own_cells_in_ext"]:
            c = lay.ext_cells[c_ext]
            assert np.array_equal(lay.ext_faces[sets[c_ext]], glob[c])
