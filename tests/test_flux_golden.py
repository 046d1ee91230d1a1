"""Pin the oracle's flux recovery / CFL / step control
against the reference's own outputs (tests/golden/make_flux_golden.py).  The
blocks and element operators come from the repo's host assembly, itself
pinned to the reference (tests/test_assembly_golden.py)."""

from __future__ import annotations

import numpy as np
import pytest

from conftest import golden
from oracle import edfa_oracle as O
from paper_2009_13916_b200 import assembly, configs, mesh


def system(name):
    if name == "config2_n6":
        n, h = 6, 1000.0 / 6
        g = mesh.box_grid(n, n, n, h, h, h)
        fld = configs.lognormal_aniso_field(g.n_elems, configs.SEEDS[2])
        bc = mesh.Boundaries(pressure_planes={"x-": 1.0, "x+": 0.0})
    else:
        n = 5
        g = mesh.perturb_interior(mesh.box_grid(n, n, n, 1 / n, 1 / n, 1 / n), 0.2, configs.SEEDS[3])
        fld = configs.rotated_tensor_field(g.n_elems, configs.SEEDS[3] + 1)
        bc = mesh.Boundaries(wells=[(0, 0, 1.0), (n - 1, n - 1, 0.0)])
    return g, fld, bc


@pytest.mark.parametrize("name", ["config2_n6", "config3_n5"])
def test_flux_cfl_balance_match_reference(name):
    d = golden("flux_" + name)
    g, fld, bc = system(name)
    s = assembly.assemble(g, fld, mesh.RockProps(gamma=1.0), bc, float(d["dt"]), d["p_prev"])
    pi, p = s.split(d["x"])
    pif = O.face_pressures(g.n_faces, s.free_faces, s.dirichlet_faces, s.dirichlet_values, pi)
    q = O.recover_face_fluxes(g.elem_to_faces, g.face_to_elems, g.face_local, s.ops.Binv, s.ops.row_sums,
                              s.ops.diag, pif, p)
    assert np.abs(q - d["q"]).max() <= 1e-12 * np.abs(d["q"]).max()
    chi = O.cfl(g.elem_to_faces, g.face_to_elems, q, g.elem_volume, d["porosity"], float(d["dt"]))
    assert np.abs(chi - d["chi"]).max() <= 1e-12 * np.abs(d["chi"]).max()
    res = O.balance_residuals(g.elem_to_faces, g.face_to_elems, q, g.elem_volume, s.accumulation,
                              float(d["dt"]), p, d["p_prev"])
    assert np.abs(res - d["balance"]).max() <= 1e-9
    dp = float(np.abs(p - d["p_prev"]).max())
    assert dp == pytest.approx(float(d["dp_max"]), rel=1e-14)
    assert O.next_dt(float(d["dt"]), 5.0, 1.1, 5.0, dp) == pytest.approx(float(d["next_dt"]), rel=1e-14)
    assert O.next_dt(float(d["dt"]), 5.0, 1.1, 5.0, 0.0) == pytest.approx(float(d["next_dt_quiet"]), rel=1e-14)
