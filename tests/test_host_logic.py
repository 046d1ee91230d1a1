"""Host-side logic of the device assembly and the transient loop that needs
no GPU: boundary resolution into per-face codes, the step controller."""

from __future__ import annotations

import numpy as np
import pytest

from oracle import edfa_oracle as O
from paper_2009_13916_b200 import mesh
from paper_2009_13916_b200.device_assembly import BC_FLUX, BC_NONE, BC_PRESSURE, face_conditions, next_dt


def test_face_conditions_codes():
    g = mesh.box_grid(4, 3, 2, 1.0, 1.0, 1.0)
    bc = mesh.Boundaries(pressure_planes={"x-": 2.0}, flux_planes={"z+": -0.5}, wells=[(3, 2, 7.0)])
    code, value, df, dv = face_conditions(g, bc)
    rdf, rdv, rnf, rnv = bc.resolve(g)
    assert np.array_equal(df, rdf) and np.array_equal(dv, rdv)
    assert (code[rdf] == BC_PRESSURE).all() and np.array_equal(value[rdf], rdv)
    assert (code[rnf] == BC_FLUX).all() and np.array_equal(value[rnf], rnv)
    rest = np.setdiff1d(np.arange(g.n_faces), np.concatenate([rdf, rnf]))
    assert (code[rest] == BC_NONE).all()


def test_face_conditions_rejects_interior_flux():
    g = mesh.box_grid(3, 3, 3, 1.0, 1.0, 1.0)

    class Interior(mesh.Boundaries):
        def resolve(self, grid):
            interior = np.flatnonzero(grid.face_to_elems[:, 1] >= 0)[:1]
            return (np.empty(0, np.int64), np.empty(0), interior, np.ones(1))

    with pytest.raises(ValueError, match="interior"):
        face_conditions(g, Interior())


@pytest.mark.parametrize("dt,dp", [(0.1, 0.0), (0.1, 1.0), (0.1, 50.0), (4.9, 0.01), (1.0, 5.0)])
def test_step_controller_matches_oracle(dt, dp):
    assert next_dt(dt, 5.0, 1.1, 5.0, dp) == O.next_dt(dt, 5.0, 1.1, 5.0, dp)


def test_matrix_market_roundtrip(tmp_path):
    """mm_write / mm_read (hx/sparse.py:302-317): 17 significant digits make
    the round trip exact; vectors come back as n x 1 canonical CSR."""
    import scipy.sparse as sp

    from paper_2009_13916_b200.sparse import canonical, mm_read, mm_write
    rng = np.random.default_rng(0)
    A = canonical(sp.random(40, 30, density=0.1, random_state=1, format="csr"))
    A.data = rng.standard_normal(A.nnz) * 10.0 ** rng.uniform(-12, 12, A.nnz)
    mm_write(A, tmp_path / "A.mtx")
    B = mm_read(tmp_path / "A.mtx")
    assert B.shape == A.shape and np.array_equal(B.indptr, A.indptr) and np.array_equal(B.indices, A.indices)
    assert np.array_equal(B.data, A.data)
    v = rng.standard_normal(17)
    mm_write(v, tmp_path / "v.mtx")
    w = mm_read(tmp_path / "v.mtx")
    assert w.shape == (17, 1) and np.array_equal(w.toarray().ravel(), v)
    S = canonical(A[:30, :30] + A[:30, :30].T)
    mm_write(S, tmp_path / "S.mtx", symmetric=True)
    assert abs(mm_read(tmp_path / "S.mtx") - S).max() == 0.0
    (tmp_path / "bad.mtx").write_text("not a matrix market file\n")
    with pytest.raises(Exception):
        mm_read(tmp_path / "bad.mtx")
