"""Pin the CPU oracle against artefacts of the unmodified reference.

tests/golden/*.npz were produced by tests/golden/make_golden.py, which runs
hexflow 0.1.0 (the reference) in the build container.  The oracle must
reproduce every one of them bit for bit: restriction sets, G, F, H, the IC
factor of -A_ff, S, its ILU factors and a preconditioner application.
"""

from __future__ import annotations

import numpy as np
import pytest

from conftest import g_blocks, g_csr, g_sets, golden, same_csr
from oracle import edfa_oracle as O

CASES = []
for _f in ("small_wells", "config1_n6", "config2_n8", "config3_n5"):
    _d = golden(_f)
    for _t in sorted({k[:-6] for k in _d if k.endswith("_G_ptr")}):
        CASES.append((_f, _t))


def options(tag):
    """Build options each golden tag was generated with (make_golden.py)."""
    s1, s2 = {"no_fill": True}, {"no_fill": True}
    dyn = None
    if tag.startswith("dyn"):
        dyn = (int(tag[3]), int(tag[4]), None)
    if tag == "base_fill":
        s1, s2 = {}, {}
    if tag == "base_thresh":
        s1, s2 = {"face_drop_tol": 1e-3}, {"schur_drop_tol": 1e-3}
    if tag == "dyn14_pre":
        s1.update(tau_filt=1e-3, filtration="pre")
    if tag == "dyn14_postprod":
        s1.update(tau_filt=0.05, filtration="post-product")
    if tag == "dyn14_postschur":
        s2.update(tau_filt=0.05, filtration="post-schur")
    return dyn, s1, s2


@pytest.mark.parametrize("fname,tag", CASES)
def test_oracle_reproduces_reference(fname, tag):
    d = golden(fname)
    A_ff, A_fc, A_cf, A_cc = g_blocks(d)
    dyn, o1, o2 = options(tag)
    Q = g_sets(d, tag + "_Q")
    s1 = O.build_stage1(A_ff, A_fc, A_cf, sets=None if dyn else Q, dynamic=dyn, **o1)
    s2 = O.build_stage2(A_cc, s1, **o2)
    assert all(np.array_equal(a, b) for a, b in zip(s1.sets, Q))
    for mine, ref in ((s1.G, "G"), (s1.F, "F"), (s1.H, "H"),
                      (s1.face_inner.L, "Lff"), (s2.S, "S"),
                      (s2.schur_inner.L, "LS"), (s2.schur_inner.U, "US")):
        R = g_csr(d, f"{tag}_{ref}")
        assert same_csr(mine, R), ref
        assert np.array_equal(mine.tocsr().data, R.data), ref
    y = O.apply(s1, s2, A_fc, A_cf, d[tag + "_apply_r"])
    assert np.array_equal(y, d[tag + "_apply_y"])
    mu = O.density(s1, s2, A_ff, A_fc, A_cf, A_cc)
    assert mu == float(d[tag + "_density"])


def test_oracle_bicgstab_matches_reference_history():
    d = golden("small_wells")
    A_ff, A_fc, A_cf, A_cc = g_blocks(d)
    s1 = O.build_stage1(A_ff, A_fc, A_cf, sets=g_sets(d, "base_nofill_Q"), no_fill=True)
    s2 = O.build_stage2(A_cc, s1, no_fill=True)
    import scipy.sparse as sp
    A = sp.bmat([[A_ff, A_fc], [A_cf, A_cc]], format="csr")
    x, rep = O.bicgstab(lambda v: A @ v, lambda r: O.apply(s1, s2, A_fc, A_cf, r),
                        d["rhs"], tol=1e-8)
    assert rep.n_it == int(d["base_nofill_bicg_nit"])
    assert np.array_equal(np.array(rep.relres_history), d["base_nofill_bicg_hist"])
    assert np.array_equal(x, d["base_nofill_bicg_x"])


def test_oracle_static_prototypes_match_reference():
    from paper_2009_13916_b200 import mesh
    d = golden("protos")
    g = mesh.box_grid(5, 5, 5, 1.0, 1.0, 1.0)
    for p in "ABCDE":
        mine = O.static_sets(g, d["face_index"], p)
        ref = g_sets(d, f"proto{p}")
        assert all(np.array_equal(a, b) for a, b in zip(mine, ref)), p


def test_oracle_gmres_basic_contracts():
    rng = np.random.default_rng(0)
    A = rng.standard_normal((30, 30)) + 30 * np.eye(30)
    b = rng.standard_normal(30)
    Ainv = np.linalg.inv(A)
    x, rep = O.gmres(lambda v: A @ v, lambda v: Ainv @ v, b, tol=1e-10)
    assert rep.converged and rep.n_it <= 2
    x, rep = O.gmres(lambda v: A @ v, None, b, tol=1e-10, restart=5)
    assert rep.converged and rep.final_relres <= 1e-10
    assert len(rep.relres_history) == rep.n_it
    x, rep = O.gmres(lambda v: A @ v, None, np.zeros(30))
    assert rep.converged and not x.any()
    with pytest.raises(ValueError):
        O.gmres(lambda v: v, None, b, tol=0.0)
