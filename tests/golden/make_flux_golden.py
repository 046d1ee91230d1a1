"""Golden artefacts of the reference's flux recovery and CFL.

Run in the build container only (needs /root/reference):

    python tests/golden/make_flux_golden.py

Writes ``tests/golden/flux_*.npz``: for a grid built with the repo's seeded
generators and assembled by the UNMODIFIED reference, a seeded solution
vector x of one backward-Euler step and the reference's
``recover_face_fluxes`` (hx/assembly.py:334-356), ``cfl`` (hx/driver.py:67-71),
``balance_residuals`` (hx/assembly.py:367-387) and ``next_dt``
(hx/driver.py:50-53) on it.
"""

from __future__ import annotations

import math
import pathlib
import sys

import numpy as np

HERE = pathlib.Path(__file__).resolve().parent
REPO = HERE.parent.parent
sys.path.insert(0, str(REPO))
sys.path.insert(0, "/root/reference/pkg/src")

import hexflow as hx                                    # noqa: E402
from hexflow.assembly import balance_residuals, recover_face_fluxes  # noqa: E402
from hexflow.driver import TimestepController, cfl, next_dt  # noqa: E402
from hexflow.grid import BoundarySpec                   # noqa: E402

from make_golden import ref_grid                        # noqa: E402
from paper_2009_13916_b200 import configs, mesh         # noqa: E402


def case(name, g_ref, tensors, bc, dt, p_prev, seed):
    fld = hx.ConductivityField(tensors)
    props = hx.FluidRockProps.uniform(g_ref.n_elems, gamma=1.0)
    s = hx.assemble(g_ref, fld, props, bc, dt=dt, p_prev=p_prev)
    A = s.full_matrix()
    rng = np.random.default_rng(seed)
    x = rng.standard_normal(s.n_unknowns) * 0.1 + 1.0
    x = np.linalg.solve(A.toarray(), s.rhs()) if s.n_unknowns < 4000 else x
    pi, p = s.split(x)
    q = recover_face_fluxes(s, pi, p)
    st = cfl(g_ref, q, props.porosity, dt)
    res = balance_residuals(s, pi, p, p_prev=p_prev)
    ctrl = TimestepController(dt=dt, dt_max=5.0, dt_mult=1.1, dp_target=5.0)
    dp = float(np.abs(p - p_prev).max())
    out = dict(x=x, q=q, chi=st.chi, balance=res, dp_max=dp, next_dt=ctrl.advance(dp),
               next_dt_quiet=next_dt(TimestepController(dt=dt, dt_max=5.0, dt_mult=1.1, dp_target=5.0)),
               dt=dt, p_prev=p_prev, porosity=props.porosity)
    np.savez_compressed(HERE / f"flux_{name}.npz", **out)
    print(name, s.n_unknowns, float(np.abs(q).max()), float(st.chi.max()))


def main():
    # config-2 generator at 6^3, transient step from p_prev = 0.5
    n = 6
    h = 1000.0 / n
    g = mesh.box_grid(n, n, n, h, h, h)
    fld = configs.lognormal_aniso_field(g.n_elems, configs.SEEDS[2])
    gr = ref_grid(n, n, n, h, h, h)
    bc = BoundarySpec().add_plane(gr, "x-", pressure=1.0).add_plane(gr, "x+", pressure=0.0)
    case("config2_n6", gr, fld.tensors, bc, 0.5, np.full(g.n_elems, 0.5), 1)
    # config-3 generator at 5^3 (distorted, full tensors, wells)
    n = 5
    g3 = mesh.perturb_interior(mesh.box_grid(n, n, n, 1 / n, 1 / n, 1 / n), 0.2, configs.SEEDS[3])
    fld3 = configs.rotated_tensor_field(g3.n_elems, configs.SEEDS[3] + 1)
    bc3 = BoundarySpec(well_columns=[(0, 0, 1.0), (n - 1, n - 1, 0.0)])
    rng = np.random.default_rng(7)
    case("config3_n5", ref_grid(n, n, n, 1 / n, 1 / n, 1 / n, g3.node_coords), fld3.tensors, bc3, 0.2,
         rng.uniform(0.2, 0.8, g3.n_elems), 2)


if __name__ == "__main__":
    main()
