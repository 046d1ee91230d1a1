"""GPU parity of the threshold inner factorisations.

IC(tau) of -A_ff and ILU(tau) of S~ with fill-in (no_fill=False) and/or a
drop tolerance -- the reference CLI's default inner solves (hx/config.py:
79-83) -- through the C ABI, against
  * the reference's own artefacts (golden ``base_fill``: complete
    factorisations, the reference's build() defaults; ``base_thresh``:
    tau = 1e-3 with fill), and
  * the pinned oracle (tests/test_oracle_golden.py) fed the GPU's own S~ at
    larger sizes, where the factors must be bit-identical: the kernels
    perform the reference's operations in the reference's order, so the
    drop decisions and every value coincide.
"""

from __future__ import annotations

import numpy as np
import pytest

from conftest import GoldenSystem, g_csr, g_sets, golden, same_csr
from oracle import edfa_oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def edfa(cuda):
    import paper_2009_13916_b200 as E
    from paper_2009_13916_b200 import _lib
    _lib.lib()
    return E


class _PS:
    def __init__(self, sets):
        self.sets = sets
        self.provenance = "golden"


def bit_identical(A, R):
    A, R = A.tocsr(), R.tocsr()
    return same_csr(A, R) and np.array_equal(A.data, R.data)


@pytest.mark.parametrize("tag,kw", [("base_fill", {}),
                                    ("base_thresh", dict(face_drop_tol=1e-3, schur_drop_tol=1e-3))])
def test_threshold_factors_match_reference(edfa, tag, kw):
    d = golden("small_wells")
    s = GoldenSystem(d)
    pre = edfa.BlockLDUPreconditioner.build(s, patterns=_PS(g_sets(d, tag + "_Q")), **kw)
    s1, s2 = pre.stage1, pre.stage2
    assert bit_identical(s1.face_inner.L, g_csr(d, tag + "_Lff")), "IC(tau) must be bit-identical"
    S_ref = g_csr(d, tag + "_S")
    assert abs(s2.S - S_ref).max() <= 1e-10 * abs(S_ref).max()
    # the ILU factors of the GPU's own S~ equal the pinned oracle's bit for bit ...
    tol = kw.get("schur_drop_tol", 0.0)
    ref = O.ilu(s2.S, tol, no_fill=False)
    assert bit_identical(s2.schur_inner.L, ref.L) and bit_identical(s2.schur_inner.U, ref.U)
    # ... and the reference's where S~ coincides in pattern
    if same_csr(s2.S, S_ref):
        for part, name in ((s2.schur_inner.L, "LS"), (s2.schur_inner.U, "US")):
            R = g_csr(d, f"{tag}_{name}")
            assert same_csr(part, R), name
            assert abs(part - R).max() <= 1e-9 * abs(R).max(), name
        y = pre.apply(d[tag + "_apply_r"])
        yr = d[tag + "_apply_y"]
        assert np.abs(y - yr).max() <= 1e-8 * np.abs(yr).max()
        assert pre.density == pytest.approx(float(d[tag + "_density"]), rel=0, abs=1e-12)
    x, rep = edfa.bicgstab(edfa.system_operator(pre.device_system), pre, s.rhs(), tol=1e-8)
    assert rep.converged and abs(rep.n_it - int(d[tag + "_bicg_nit"])) <= 2


CASES = [(2, 10, "static"), (3, 6, "static"), (3, 5, "dynamic"), (1, 9, "base"), (4, 0, "static")]


def _case(idx, n):
    from paper_2009_13916_b200 import configs
    if idx == 4:
        return configs.config4(nx=6, ny=9, nz=5)
    return configs.make(idx, n=n)


def _build(E, s, kind, **kw):
    if kind == "dynamic":
        return E.BlockLDUPreconditioner.build(s, dynamic=E.DynamicConfig(1, 4), **kw)
    pats = E.patterns_for(s, kind, "A") if kind != "base" else E.patterns_for(s, "base")
    return E.BlockLDUPreconditioner.build(s, patterns=pats, **kw)


@pytest.mark.parametrize("idx,n,kind", CASES)
@pytest.mark.parametrize("tol,no_fill", [(1e-3, False), (1e-2, False), (1e-3, True)])
def test_threshold_factors_match_oracle(edfa, idx, n, kind, tol, no_fill):
    s = _case(idx, n).system
    pre = _build(edfa, s, kind, face_drop_tol=tol, schur_drop_tol=tol, no_fill=no_fill)
    s1, s2 = pre.stage1, pre.stage2
    ic_ref = O.ic(-s.A_ff, tol, no_fill=no_fill)
    assert bit_identical(s1.face_inner.L, ic_ref.L), "IC(tau) differs from the oracle"
    assert s1.face_inner.pivot_shifts == ic_ref.pivot_shifts
    ilu_ref = O.ilu(s2.S, tol, no_fill=no_fill)
    assert bit_identical(s2.schur_inner.L, ilu_ref.L), "ILU(tau) L differs from the oracle"
    assert bit_identical(s2.schur_inner.U, ilu_ref.U), "ILU(tau) U differs from the oracle"
    assert s2.schur_inner.nnz_stored == ilu_ref.nnz_stored
    assert s1.face_inner.nnz_stored == ic_ref.nnz_stored
    # the inner solves apply the factors: (L U)^-1 r against scipy's triangular solves
    r = np.random.default_rng(3).standard_normal(s.n_cells)
    y = s2.schur_inner.apply(r)
    y_ref = ilu_ref.apply(r)
    assert np.abs(y - y_ref).max() <= 1e-10 * np.abs(y_ref).max()


@pytest.mark.parametrize("idx,n,kind", [(2, 12, "static"), (3, 6, "dynamic")])
def test_gmres_with_threshold_inner_solves(edfa, idx, n, kind):
    case = _case(idx, n)
    s = case.system
    pre = _build(edfa, s, kind, face_drop_tol=1e-3, schur_drop_tol=1e-3)
    x, rep = edfa.gmres(edfa.system_operator(pre.device_system), pre, s.rhs(), tol=1e-8, restart=50)
    A = s.full_matrix()
    b = s.rhs()
    x = x.cpu().numpy() if hasattr(x, "cpu") else x
    assert rep.converged and np.linalg.norm(b - A @ x) <= 1e-8 * np.linalg.norm(b)
    # oracle: same stage 1 restatement with the same inner-solve options
    sets = O.static_sets(s.grid, s.face_index, "A") if kind == "static" else None
    o1 = O.build_stage1(s.A_ff, s.A_fc, s.A_cf, sets=sets, dynamic=None if sets is not None else (1, 4, None),
                        face_drop_tol=1e-3)
    o2 = O.build_stage2(s.A_cc, o1, schur_drop_tol=1e-3)
    xo, ro = O.gmres(lambda v: A @ v, lambda r: O.apply(o1, o2, s.A_fc, s.A_cf, r), b, tol=1e-8, restart=50)
    assert abs(rep.n_it - ro.n_it) <= 2
    assert np.linalg.norm(x - xo) <= 1e-7 * np.linalg.norm(xo)


def test_threshold_overflow_is_reported(edfa):
    """A complete factorisation whose rows outgrow the working table fails
    loudly (EdfaUnsupported), never silently approximates."""
    import ctypes as C

    import scipy.sparse as sp

    from paper_2009_13916_b200 import _lib as L
    from paper_2009_13916_b200.device import DeviceCsr, ctx
    n = 4000                                              # arrow: the last row holds n entries
    M = sp.lil_matrix((n, n))
    M.setdiag(4.0)
    M[n - 1, :] = 1.0
    M[n - 1, n - 1] = 4.0 * n
    A = DeviceCsr.from_scipy(sp.csr_matrix(M))
    f = C.c_void_p()
    with pytest.raises(L.EdfaUnsupported):
        L.check(L.lib().edfa_factor_ilu(ctx(), A.handle, 0.0, 0, 0, 0, 0, C.byref(f)))
    rng = np.random.default_rng(0)
    M = rng.standard_normal((600, 600)) + 600 * np.eye(600)
    # the same matrix with a drop tolerance that keeps rows short factorises
    B = sp.csr_matrix(np.where(np.abs(M) > 2.5, M, 0.0))
    Bd = DeviceCsr.from_scipy(B)
    L.check(L.lib().edfa_factor_ilu(ctx(), Bd.handle, 0.5, 0, 0, 0, 0, C.byref(f)))
    L.lib().edfa_factor_destroy(f)


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_csr_sub_matches_scipy_bitwise(edfa, seed):
    """S = A - H (hx/precond.py:264-271, tau = 0) on the eight-lanes-per-row
    kernel: pattern and values bit-identical to scipy's canonical difference,
    exact zeros dropped; covers empty rows, rows of A wider than the lane group,
    unions wider than the shared-memory mask, and cancelling entries."""
    import ctypes as C
    import scipy.sparse as sp
    from paper_2009_13916_b200 import _lib as L
    from paper_2009_13916_b200.device import DeviceCsr, ctx
    rng = np.random.default_rng(seed)
    n = 3000
    def rand(widths):
        rows, cols = [], []
        for i, w in enumerate(widths):
            c = rng.choice(n, size=int(w), replace=False)
            rows += [i] * int(w)
            cols += c.tolist()
        M = sp.csr_matrix((rng.standard_normal(len(rows)), (rows, cols)), shape=(n, n))
        M.sort_indices()
        return M
    wa = rng.choice([0, 1, 1, 1, 3, 7, 8, 9, 20], size=n)
    wh = rng.choice([0, 5, 18, 37, 37, 60, 125, 140], size=n)
    A, H = rand(wa), rand(wh)
    # cancelling entries: copy some of A's values into H at shared columns
    H = H.tolil()
    Ac = A.tocoo()
    pick = rng.random(Ac.nnz) < 0.3
    for i, j, v in zip(Ac.row[pick], Ac.col[pick], Ac.data[pick]):
        H[i, j] = v
    H = H.tocsr()
    H.sort_indices()
    ref = (A - H).tocsr()
    ref.eliminate_zeros()
    ref.sort_indices()
    dA, dH = DeviceCsr.from_scipy(A), DeviceCsr.from_scipy(H)
    h = C.c_void_p()
    L.check(L.lib().edfa_csr_sub(ctx(), dA.handle, dH.handle, 0.0, C.byref(h)))
    S = DeviceCsr(h).to_scipy()
    assert bit_identical(S, ref)
