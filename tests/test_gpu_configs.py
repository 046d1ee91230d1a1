"""BASELINE configs 3 and 4 with their bench options against the pinned oracle.

Fixtures come from tests/golden/make_oracle_configs.py (the oracle port run on
the same seeded generators at CPU-feasible sizes).  Gates (BASELINE
north_star): restriction sets bit-exact and G~/F~ rows within 1e-10 relative
on a seeded sample of cells, GMRES(50) iterations within 2 of the oracle's,
final true relative residual <= rtol, solution within 1e-7 relative.
"""

from __future__ import annotations

import numpy as np
import pytest

from conftest import golden

pytestmark = pytest.mark.gpu

CASES = {
    "c3_24": lambda c: c.config3(n=24),
    "c3_32": lambda c: c.config3(n=32),
    "c4": lambda c: c.config4(nx=20, ny=73, nz=28),
}


@pytest.fixture(scope="module")
def edfa(cuda):
    import paper_2009_13916_b200 as E
    return E


def build(edfa, case, ds):
    """The bench's preconditioner for a config (configs.py options; the
    face and Schur factorisations may differ in fill, as the stage-level
    reference API allows)."""
    p = case.precond
    face_nf = p.get("face_no_fill", p.get("no_fill", True))
    schur_nf = p.get("schur_no_fill", p.get("no_fill", True))
    kw = dict(face_drop_tol=p.get("face_drop_tol", 0.0), no_fill=face_nf)
    if p["pattern"] == "dynamic":
        s1 = edfa.build_stage1(ds, dynamic=edfa.DynamicConfig(p["n_add"], p["n_ent"]), **kw)
    else:
        s1 = edfa.build_stage1(ds, patterns=edfa.patterns_for(ds, p["pattern"], p.get("prototype", "A")), **kw)
    pre = edfa.BlockLDUPreconditioner(ds, s1, settings=dict(tau_filt=0.0, filtration="none",
                                                             schur_drop_tol=p.get("schur_drop_tol", 0.0),
                                                             no_fill=schur_nf))
    pre.refresh(ds)
    return pre


def rows_of(d, name, k):
    p = d[name + "_ptr"]
    return slice(int(p[k]), int(p[k + 1]))


@pytest.mark.parametrize("name", sorted(CASES))
def test_config_matches_oracle_fixture(edfa, name):
    from paper_2009_13916_b200 import configs
    d = golden(f"oracle_{name}")
    case = CASES[name](configs)
    s = case.system
    ds = edfa.DeviceSystem.from_host(s)
    pre = build(edfa, case, ds)
    # stage 1 on the sampled cells: sets bit-exact, G~ / F~ rows <= 1e-10 relative
    sets = pre.stage1.patterns.sets
    G, FT = pre.stage1.G, pre.stage1.F.T.tocsr()
    for k, m in enumerate(d["rows"]):
        assert np.array_equal(np.asarray(sets[m], dtype=np.int64), d["set_idx"][rows_of(d, "set", k)]), m
        for M, nm in ((G, "G"), (FT, "F")):
            lo, hi = M.indptr[m], M.indptr[m + 1]
            ri, rv = d[nm + "_idx"][rows_of(d, nm, k)], d[nm + "_val"][rows_of(d, nm, k)]
            assert np.array_equal(M.indices[lo:hi], ri), (nm, m)
            assert np.abs(M.data[lo:hi] - rv).max(initial=0.0) <= 1e-10 * np.abs(rv).max(initial=1.0), (nm, m)
    # H~ / S~ sizes: equal up to roundoff-size entries on either side
    for got, want in ((pre.stage1.H.nnz, int(d["nnz_H"])), (pre.stage2.S.nnz, int(d["nnz_S"]))):
        assert abs(got - want) <= 1e-4 * want, (got, want)
    x, rep = edfa.gmres(edfa.system_operator(ds), pre, s.rhs(), tol=case.rtol, restart=case.restart,
                        max_it=case.max_it)
    assert bool(d["converged"]) and rep.converged
    assert abs(rep.n_it - int(d["n_it"])) <= 2, (rep.n_it, int(d["n_it"]))
    A, b = s.full_matrix(), s.rhs()
    assert np.linalg.norm(b - A @ x) <= case.rtol * np.linalg.norm(b) * 1.0001
    assert abs(np.linalg.norm(x) - float(d["x_norm"])) <= 1e-7 * float(d["x_norm"])
    assert np.abs(x[::37] - d["x_sub"]).max() <= 1e-7 * np.abs(d["x_sub"]).max()


def test_config5_sample_matches_oracle(edfa):
    """BASELINE config 5 (256^3) gated on samples: the full
    system is assembled and its stage 1 built on the GPU; the restriction sets
    and G~/F~ rows of 10,240 seeded random cells equal the oracle's (sets
    bit-exact, rows <= 1e-10); the GPU ILU(0) of the oracle's S~ sub-block (a
    64 x 64 patch of one cell layer) reproduces the oracle's factors bit for
    bit."""
    import scipy.sparse as sp

    from paper_2009_13916_b200 import configs
    from paper_2009_13916_b200 import device_assembly as DA
    from paper_2009_13916_b200.parallel import _sub_face_keys
    d = golden("oracle_c5_sample")
    n = 256
    case = configs.inputs_only(5, n=n)
    dsys = DA.assemble_device(*case.meta["inputs"], element_ops=False)
    ds = dsys.system
    s1 = edfa.build_stage1(ds, patterns=edfa.patterns_for(ds, "static", "A"), no_fill=True)
    fidx = dsys.face_index.cpu().numpy()
    gkey, _ = _sub_face_keys(n, n, n, 0, n)
    free_gid = gkey[np.flatnonzero(fidx >= 0)]                  # free index -> global face id
    rows = d["rows"]
    sets = s1.patterns                                           # device pattern, exported once
    Qp, Qi, _ = sets._dev.arrays(values=False)
    G = s1.G
    FT = s1.F.T.tocsr()
    for k, m in enumerate(rows):
        q = free_gid[Qi[Qp[m]:Qp[m + 1]]]
        assert np.array_equal(q, d["set_idx"][rows_of(d, "set", k)]), m
        for M, nm in ((G, "G"), (FT, "F")):
            lo, hi = M.indptr[m], M.indptr[m + 1]
            ri, rv = d[nm + "_idx"][rows_of(d, nm, k)], d[nm + "_val"][rows_of(d, nm, k)]
            assert np.array_equal(free_gid[M.indices[lo:hi]], ri), (nm, m)
            assert np.abs(M.data[lo:hi] - rv).max(initial=0.0) <= 1e-10 * np.abs(rv).max(initial=1.0), (nm, m)
    del s1, G, FT
    ns = int(d["S_n"])
    S = sp.csr_matrix((d["S_val"], d["S_idx"], d["S_ptr"]), shape=(ns, ns))
    import ctypes as C

    from paper_2009_13916_b200 import _lib as L
    from paper_2009_13916_b200.device import DeviceCsr, ctx
    Sd = DeviceCsr.from_scipy(S)
    f = C.c_void_p()
    L.check(L.lib().edfa_factor_ilu(ctx(), Sd.handle, 0.0, 1, 0, 0, 0, C.byref(f)))
    parts = []
    for which in (0, 1):
        h = C.c_void_p()
        L.check(L.lib().edfa_factor_part(ctx(), f, which, C.byref(h)))
        parts.append(DeviceCsr(h, owner=False).to_scipy())
    L.lib().edfa_factor_destroy(f)
    for M, nm in ((parts[0], "L"), (parts[1], "U")):
        assert np.array_equal(M.indptr, d[nm + "_ptr"]) and np.array_equal(M.indices, d[nm + "_idx"]), nm
        assert np.array_equal(M.data, d[nm + "_val"]), nm


def test_config4_stagnation_matches_oracle(edfa):
    """Config 4 does not reach rtol at its BASELINE size with any
    reference-native option (GMRES(50) stalls at relres
    ~1e-5..1e-4 after 2000 iterations); the pinned oracle shows the same
    stall on the largest CPU-feasible box (30 x 110 x 42, bench options,
    600 iterations).  The GPU solve of the same system follows the oracle's
    residual history: both stall, at the same level within a factor 2."""
    from paper_2009_13916_b200 import configs
    d = golden("oracle_c4_30")
    case = configs.config4(nx=30, ny=110, nz=42)
    s = case.system
    ds = edfa.DeviceSystem.from_host(s)
    pre = build(edfa, case, ds)
    max_it = int(d["max_it"])
    x, rep = edfa.gmres(edfa.system_operator(ds), pre, s.rhs(), tol=case.rtol, restart=case.restart,
                        max_it=max_it)
    h_gpu, h_ref = np.array(rep.relres_history), d["hist"]
    assert not bool(d["converged"]) and not rep.converged and rep.n_it == int(d["n_it"]) == max_it
    for it in (100, 300, max_it - 1):
        assert 0.5 <= h_gpu[it] / h_ref[it] <= 2.0, (it, h_gpu[it], h_ref[it])
    assert 0.5 <= rep.final_relres / float(d["final_relres"]) <= 2.0
