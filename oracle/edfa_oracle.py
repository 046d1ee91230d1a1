"""CPU restatement of the EDFA preconditioner path -- TEST INFRASTRUCTURE ONLY.

Never imported by the product package.  Each function cites the reference
(hexflow 0.1.0 under /root/reference/pkg/src/hexflow, abbreviated ``hx/``)
file:line it restates.  The arithmetic that lives in third-party native code
is delegated to the same third-party code the reference calls:

* dense SPD solves: ``scipy.linalg.cho_factor/cho_solve`` (LAPACK potrf/potrs
  from scipy-openblas 0.3.31, scipy 1.18.1), call site hx/sparse.py:95-98;
* sparse products: scipy sparsetools ``csr_matmat`` (hx/precond.py:257);
* triangular solves: ``scipy.sparse.linalg.spsolve_triangular``
  (hx/sparse.py:127-129).

Incomplete factorizations (hx/sparse.py:141-282) are pure Python in the
reference and are restated here operation-for-operation (same update order,
no fused multiply-add) so that the oracle reproduces the reference bit for
bit; ``tests/test_oracle_golden.py`` pins that against reference-generated
golden files.
"""

from __future__ import annotations

import bisect
import math

import numpy as np
import scipy.linalg
import scipy.sparse as sp
from scipy.sparse.linalg import spsolve_triangular

PIVOT_GUARD = 1e-12                       # hx/sparse.py:24-25
FILTRATION_MODES = ("none", "pre", "post-schur", "post-product")  # hx/precond.py:35


class OracleFactorizationError(RuntimeError):
    """Dense Cholesky failure (hx/errors.py:16; raised at hx/sparse.py:94-97)."""


def canonical(A) -> sp.csr_matrix:
    """hx/sparse.py:28-34: sorted, duplicates summed, explicit zeros dropped."""
    A = sp.csr_matrix(A, copy=True)
    A.sum_duplicates()
    A.sort_indices()
    A.eliminate_zeros()
    return A


# ---------------------------------------------------------------------------
# restriction patterns (hx/patterns.py)

def base_sets(A_cf: sp.csr_matrix):
    """hx/patterns.py:55-60 -- column pattern of each A_cf row."""
    A = A_cf.tocsr()
    return [np.sort(A.indices[A.indptr[m]:A.indptr[m + 1]].astype(np.int64))
            for m in range(A.shape[0])]


def _nbr(grid, e, slot):
    a, b = grid.face_to_elems[grid.elem_to_faces[e, slot]]
    return int(b if a == e else a)


def static_set(grid, proto: str, m: int) -> np.ndarray:
    """hx/patterns.py:63-121 -- geometric prototype patch around cell m."""
    if proto not in "ABCDE" or len(proto) != 1:
        raise ValueError(f"unknown prototype {proto!r}")
    e2f = grid.elem_to_faces
    out = set(int(f) for f in e2f[m])

    def chain(slot, depth):
        cur = m
        for _ in range(depth):
            cur = _nbr(grid, cur, slot)
            if cur < 0:
                return
            out.add(int(e2f[cur, slot]))

    if proto in "ABE":
        for slot in range(6):
            chain(slot, {"A": 2, "B": 3, "E": 1}[proto])
        if proto == "E":
            for slot in range(6):
                nb = _nbr(grid, m, slot)
                if nb >= 0:
                    ax, sg = divmod(slot, 2)
                    out.add(int(e2f[nb, 2 * ((ax + 1) % 3) + sg]))
    else:
        for slot in range(6):
            nb = _nbr(grid, m, slot)
            if nb >= 0:
                out.update(int(f) for f in e2f[nb])
        if proto == "D":
            for slot in range(6):
                chain(slot, 2)
    return np.array(sorted(out), dtype=np.int64)


def static_sets(grid, face_index, proto):
    """hx/patterns.py:124-133 -- prototypes in free-face numbering."""
    out = []
    for m in range(grid.elem_to_faces.shape[0]):
        red = face_index[static_set(grid, proto, m)]
        out.append(np.sort(red[red >= 0]))
    return out


# ---------------------------------------------------------------------------
# restricted solves and dynamic growth (hx/precond.py:70-135)

def principal_submatrix(A: sp.csr_matrix, idx) -> np.ndarray:
    """Dense A[idx, idx] (hx/sparse.py:61-84)."""
    idx = np.asarray(idx, dtype=np.int64)
    s = idx.size
    out = np.zeros((s, s))
    pos = {int(c): p for p, c in enumerate(idx)}
    for p, r in enumerate(idx):
        lo, hi = A.indptr[r], A.indptr[r + 1]
        for c, v in zip(A.indices[lo:hi], A.data[lo:hi]):
            q = pos.get(int(c))
            if q is not None:
                out[p, q] = v
    return out


def spd_solve(M, b):
    """hx/sparse.py:87-98: Cholesky via LAPACK, failure -> error."""
    try:
        c = scipy.linalg.cho_factor(M, check_finite=False)
    except scipy.linalg.LinAlgError as exc:
        raise OracleFactorizationError(f"dense Cholesky failed: {exc}") from exc
    return scipy.linalg.cho_solve(c, b, check_finite=False)


def restricted_solve(A_ff, rhs_idx, rhs_val, idx):
    """hx/precond.py:85-93: solve -A_ff[idx,idx] x = rhs|_idx (entries of the
    sparse rhs outside idx are dropped)."""
    idx = np.asarray(idx, dtype=np.int64)
    sub = principal_submatrix(A_ff, idx)
    b = np.zeros(idx.size)
    where = {int(c): p for p, c in enumerate(idx)}
    for c, v in zip(np.asarray(rhs_idx), np.asarray(rhs_val)):
        p = where.get(int(c))
        if p is not None:
            b[p] = v
    return spd_solve(-sub, b)


def solve_restricted_row(A_ff, rhs, idx):
    """hx/precond.py:70-82 -- dense rhs, prolonged full-length result."""
    n = A_ff.shape[0]
    out = np.zeros(n)
    idx = np.asarray(idx, dtype=np.int64)
    if idx.size:
        out[idx] = spd_solve(-principal_submatrix(A_ff, idx), np.asarray(rhs)[idx])
    return out


def prolonged_residual(A_csc, rhs_idx, rhs_val, idx, x):
    """hx/precond.py:96-104: r = rhs + A_ff R^T x on the touched support; the
    column contributions are accumulated in storage order (np.add.at)."""
    touched_rows, contrib = [], []
    for p, j in enumerate(idx):
        lo, hi = A_csc.indptr[j], A_csc.indptr[j + 1]
        touched_rows.append(A_csc.indices[lo:hi].astype(np.int64))
        contrib.append(A_csc.data[lo:hi] * x[p])
    rows = np.concatenate(touched_rows) if touched_rows else np.empty(0, np.int64)
    vals = np.concatenate(contrib) if contrib else np.empty(0)
    cand = np.unique(np.concatenate([np.asarray(rhs_idx, np.int64), rows]))
    r = np.zeros(cand.size)
    r[np.searchsorted(cand, rhs_idx)] = rhs_val
    np.add.at(r, np.searchsorted(cand, rows), vals)
    return cand, r


def sweep_limit(n_ent, it_max):
    """hx/precond.py:65-67."""
    return it_max if it_max is not None else max(n_ent, 1)


def grow_dynamic(A_ff, rhs_idx, rhs_val, n_add, n_ent, it_max=None, A_csc=None):
    """hx/precond.py:107-135 (Algorithm 1 dynamic branch)."""
    if A_csc is None:
        A_csc = A_ff.tocsc()
    rhs_idx = np.asarray(rhs_idx, dtype=np.int64)
    idx = np.unique(rhs_idx)
    x = restricted_solve(A_ff, rhs_idx, rhs_val, idx)
    added, sweeps = 0, 0
    while added < n_ent and sweeps < sweep_limit(n_ent, it_max):
        sweeps += 1
        budget = min(n_add, n_ent - added)
        cand, r = prolonged_residual(A_csc, rhs_idx, rhs_val, idx, x)
        fresh = ~np.isin(cand, idx)
        new, mag = cand[fresh], np.abs(r[fresh])
        new, mag = new[mag > 0], mag[mag > 0]
        if new.size == 0:
            break
        pick = np.lexsort((new, -mag))[:budget]       # |r| desc, index asc
        idx = np.sort(np.concatenate([idx, new[pick]]))
        added += pick.size
        x = restricted_solve(A_ff, rhs_idx, rhs_val, idx)
    return idx, x


def filter_vector(v, tau):
    """hx/precond.py:160-165."""
    if tau <= 0:
        return v
    out = v.copy()
    out[np.abs(out) < tau * np.linalg.norm(out)] = 0.0
    return out


def filter_rows(M, tau, keep_diagonal=True):
    """hx/precond.py:138-157: drop |v| < tau*||row||_2, diagonal survives."""
    if tau <= 0:
        return M
    M = canonical(M)
    for i in range(M.shape[0]):
        lo, hi = M.indptr[i], M.indptr[i + 1]
        if lo == hi:
            continue
        v = M.data[lo:hi]
        small = np.abs(v) < tau * np.linalg.norm(v)
        if keep_diagonal:
            small &= M.indices[lo:hi] != i
        v[small] = 0.0
    M.eliminate_zeros()
    return M


# ---------------------------------------------------------------------------
# incomplete factorizations (hx/sparse.py:101-282)

class Factor:
    """hx/sparse.py:101-131: kind "ilu" (unit L, U) or "ic" (L, L^T)."""

    def __init__(self, kind, L, U, shifts):
        self.kind, self.L, self.U, self.pivot_shifts = kind, L, U, shifts

    @property
    def nnz_stored(self):
        n = self.L.shape[0]
        return self.L.nnz - n + self.U.nnz if self.kind == "ilu" else 2 * self.L.nnz - n

    def apply(self, r):
        y = spsolve_triangular(self.L, r, lower=True, unit_diagonal=self.kind == "ilu")
        return spsolve_triangular(self.U, y, lower=False)


def _csr_from_rows(rows, n):
    ptr = np.zeros(n + 1, dtype=np.int32)
    cols, vals = [], []
    for i, (c, v) in enumerate(rows):
        cols.extend(c)
        vals.extend(v)
        ptr[i + 1] = len(cols)
    return sp.csr_matrix((np.array(vals, dtype=float), np.array(cols, dtype=np.int32),
                          ptr), shape=(n, n))


def ilu(A, fill_tol, no_fill=False):
    """hx/sparse.py:141-214 -- row-wise IKJ threshold ILU; pivots processed in
    increasing column order; drop on the unscaled working value; the
    sign-preserving guard replaces |pivot| < 1e-12*||row||_inf."""
    A = canonical(A)
    n = A.shape[0]
    if A.shape[1] != n:
        raise ValueError("matrix must be square")
    if fill_tol < 0:
        raise ValueError("fill_tol must be >= 0")
    ucols, uvals, diag = [None] * n, [None] * n, np.empty(n)
    lrows = []
    shifts = 0
    for i in range(n):
        lo, hi = A.indptr[i], A.indptr[i + 1]
        cols = A.indices[lo:hi].tolist()
        vals = A.data[lo:hi].tolist()
        work = dict(zip(cols, vals))
        scale = max(abs(v) for v in vals) if vals else 1.0
        tau = fill_tol * scale
        allowed = set(cols) if no_fill else None
        pending = sorted(c for c in cols if c < i)
        queued = set(pending)
        lc, lv = [], []
        while pending:
            k = pending.pop(0)
            a = work.pop(k)
            if abs(a) < tau:
                continue
            mult = a / diag[k]
            for j, u in zip(ucols[k], uvals[k]):
                if allowed is not None and j not in allowed:
                    continue
                if j in work:
                    work[j] -= mult * u
                else:
                    work[j] = -mult * u
                    if j < i and j not in queued:
                        bisect.insort(pending, j)
                        queued.add(j)
            lc.append(k)
            lv.append(mult)
        piv = work.pop(i, 0.0)
        if abs(piv) < PIVOT_GUARD * scale:
            piv = math.copysign(PIVOT_GUARD * scale, 1.0 if piv >= 0 else -1.0)
            shifts += 1
        keep = sorted((j, v) for j, v in work.items() if j > i and abs(v) >= tau)
        ucols[i] = [j for j, _ in keep]
        uvals[i] = [v for _, v in keep]
        diag[i] = piv
        lrows.append((lc + [i], lv + [1.0]))
    L = _csr_from_rows(lrows, n)
    U = _csr_from_rows(((([i] + ucols[i]), ([diag[i]] + uvals[i])) for i in range(n)), n)
    return Factor("ilu", L, U, shifts)


def ic(A, fill_tol, no_fill=False):
    """hx/sparse.py:217-282 -- up-looking threshold IC of an SPD matrix; the
    same drop/guard conventions as :func:`ilu`; returns L and L^T."""
    A = canonical(A)
    n = A.shape[0]
    if A.shape[1] != n:
        raise ValueError("matrix must be square")
    colk = [[] for _ in range(n)]        # entries (row j, L_jk) of column k
    Lrows = []
    shifts = 0
    for i in range(n):
        lo, hi = A.indptr[i], A.indptr[i + 1]
        cols = A.indices[lo:hi]
        vals = A.data[lo:hi]
        scale = float(np.abs(vals).max()) if vals.size else 1.0
        tau = fill_tol * scale
        sel = cols <= i
        work = dict(zip(cols[sel].tolist(), vals[sel].tolist()))
        allowed = set(cols[sel].tolist()) if no_fill else None
        pending = sorted(c for c in work if c < i)
        queued = set(pending)
        lc, lv = [], []
        while pending:
            k = pending.pop(0)
            wv = work.pop(k)
            if abs(wv) < tau:
                continue
            mult = wv / Lrows[k][1][-1]
            for j, ljk in colk[k]:
                if j <= k or j >= i:
                    continue
                if allowed is not None and j not in allowed:
                    continue
                if j in work:
                    work[j] -= mult * ljk
                else:
                    work[j] = -mult * ljk
                    if j not in queued:
                        bisect.insort(pending, j)
                        queued.add(j)
            work[i] = work.get(i, 0.0) - mult * mult
            lc.append(k)
            lv.append(mult)
        d = work.get(i, 0.0)
        if d < PIVOT_GUARD * scale:
            d = PIVOT_GUARD * scale
            shifts += 1
        lc.append(i)
        lv.append(float(np.sqrt(d)))
        order = np.argsort(lc)
        rc = [lc[t] for t in order]
        rv = [lv[t] for t in order]
        Lrows.append((rc, rv))
        for j, v in zip(rc[:-1], rv[:-1]):
            colk[j].append((i, v))
    L = _csr_from_rows(Lrows, n)
    return Factor("ic", L, L.T.tocsr(), shifts)


# ---------------------------------------------------------------------------
# two-stage build, application, density (hx/precond.py:168-350)

class Stage1:
    def __init__(self, G, F, H, face_inner, sizes, sets):
        self.G, self.F, self.H = G, F, H
        self.face_inner, self.pattern_sizes, self.sets = face_inner, sizes, sets


class Stage2:
    def __init__(self, S, schur_inner):
        self.S, self.schur_inner = S, schur_inner


_ROWS_CTX = {}


def _stage1_rows(m0, m1):
    """Per-cell loop of hx/precond.py:187-201 over cells [m0, m1)."""
    A_ff, A_cf, A_csc, A_fc_csc, sets, dynamic, pre_tau = (_ROWS_CTX[k] for k in (
        "A_ff", "A_cf", "A_csc", "A_fc_csc", "sets", "dynamic", "pre_tau"))
    rows, cols, gv, fv, sizes, used = [], [], [], [], [], []
    for m in range(m0, m1):
        lo, hi = A_cf.indptr[m], A_cf.indptr[m + 1]
        gi, gval = A_cf.indices[lo:hi].astype(np.int64), A_cf.data[lo:hi]
        if dynamic is not None:
            n_add, n_ent, it_max = dynamic
            idx, g = grow_dynamic(A_ff, gi, gval, n_add, n_ent, it_max, A_csc)
        else:
            idx = np.asarray(sets[m], dtype=np.int64)
            g = restricted_solve(A_ff, gi, gval, idx)
        lo, hi = A_fc_csc.indptr[m], A_fc_csc.indptr[m + 1]
        f = restricted_solve(A_ff, A_fc_csc.indices[lo:hi].astype(np.int64),
                             A_fc_csc.data[lo:hi], idx)
        rows.append(np.full(idx.size, m, dtype=np.int64))
        cols.append(idx)
        gv.append(filter_vector(g, pre_tau))
        fv.append(filter_vector(f, pre_tau))
        sizes.append(idx.size)
        used.append(idx)
    return rows, cols, gv, fv, sizes, used


def build_stage1(A_ff, A_fc, A_cf, *, sets=None, dynamic=None, tau_filt=0.0,
                 filtration="none", face_drop_tol=0.0, no_fill=False, n_workers=1):
    """hx/precond.py:187-261.  The reference fans the per-cell loop out over
    ``n_workers`` and merges in cell order (hx/precond.py:233-256), so the
    result is the serial one for any worker count; here the workers are
    processes (the reference's threads are GIL-bound).  ``dynamic`` =
    (n_add, n_ent, it_max) or None."""
    if (sets is None) == (dynamic is None):
        raise ValueError("give exactly one of patterns or dynamic")
    if filtration not in FILTRATION_MODES:
        raise ValueError(f"filtration must be one of {FILTRATION_MODES}")
    A_ff, A_cf, A_fc = canonical(A_ff), canonical(A_cf), canonical(A_fc)
    n_c, n_f = A_cf.shape[0], A_ff.shape[0]
    _ROWS_CTX.update(A_ff=A_ff, A_cf=A_cf, A_csc=A_ff.tocsc(), A_fc_csc=A_fc.tocsc(), sets=sets,
                     dynamic=dynamic, pre_tau=tau_filt if filtration == "pre" else 0.0)
    if n_workers > 1 and n_c > 1:
        import multiprocessing as mp
        cuts = np.linspace(0, n_c, n_workers + 1).astype(int)
        with mp.get_context("fork").Pool(n_workers) as pool:
            parts = pool.starmap(_stage1_rows, [(int(a), int(b)) for a, b in zip(cuts[:-1], cuts[1:])])
    else:
        parts = [_stage1_rows(0, n_c)]
    _ROWS_CTX.clear()
    rows, cols, gv, fv, sizes, used = ([x for p in parts for x in p[k]] for k in range(6))
    r = np.concatenate(rows) if rows else np.empty(0, np.int64)
    c = np.concatenate(cols) if cols else np.empty(0, np.int64)
    G = canonical(sp.coo_matrix((np.concatenate(gv) if gv else [], (r, c)), shape=(n_c, n_f)))
    F = canonical(sp.coo_matrix((np.concatenate(fv) if fv else [], (c, r)), shape=(n_f, n_c)))
    H = canonical(G @ A_ff @ F)
    if filtration == "post-product":
        H = filter_rows(H, tau_filt)
    face_inner = ic(-A_ff, face_drop_tol, no_fill=no_fill)
    return Stage1(G, F, H, face_inner, np.array(sizes), used)


def build_stage2(A_cc, stage1, *, tau_filt=0.0, filtration="none",
                 schur_drop_tol=0.0, no_fill=False):
    """hx/precond.py:264-271 (Algorithm 2)."""
    S = canonical(A_cc - stage1.H)
    if filtration == "post-schur":
        S = filter_rows(S, tau_filt)
    return Stage2(S, ilu(S, schur_drop_tol, no_fill=no_fill))


def apply(stage1, stage2, A_fc, A_cf, r):
    """hx/precond.py:311-320 -- block-triangular factored inverse."""
    n_f = A_fc.shape[0]
    r_f, r_c = r[:n_f], r[n_f:]
    t_f = -stage1.face_inner.apply(r_f)
    t_c = stage2.schur_inner.apply(r_c - A_cf @ t_f)
    y_f = t_f + stage1.face_inner.apply(A_fc @ t_c)
    return np.concatenate([y_f, t_c])


def density(stage1, stage2, A_ff, A_fc, A_cf, A_cc):
    """hx/precond.py:343-350."""
    num = (stage1.face_inner.nnz_stored + A_fc.nnz + A_cf.nnz
           + stage2.schur_inner.nnz_stored)
    return num / (A_ff.nnz + A_fc.nnz + A_cf.nnz + A_cc.nnz)


# ---------------------------------------------------------------------------
# Krylov solvers

class Report:
    """Field names of hx/krylov.py:15-37 SolveReport."""

    def __init__(self):
        self.n_it, self.converged, self.breakdown = 0, False, False
        self.relres_history, self.final_relres = [], math.inf


def bicgstab(A_apply, P_apply, b, tol=1e-8, max_it=2000):
    """hx/krylov.py:40-115 -- right-preconditioned Bi-CGStab, x0 = 0."""
    if tol <= 0:
        raise ValueError("tol must be positive")
    P_apply = P_apply or (lambda v: v)
    b = np.asarray(b, float)
    rep = Report()
    bn = np.linalg.norm(b)
    if bn == 0.0:
        rep.converged, rep.final_relres = True, 0.0
        rep.relres_history.append(0.0)
        return np.zeros_like(b), rep
    x = np.zeros_like(b)
    r = b.copy()
    rh = r.copy()
    rho = alpha = omega = 1.0
    p = np.zeros_like(b)
    v = np.zeros_like(b)
    while rep.n_it < max_it:
        rho_new = rh @ r
        if rho_new == 0.0:
            rep.breakdown = True
            break
        beta = (rho_new / rho) * (alpha / omega)
        rho = rho_new
        p = r + beta * (p - omega * v)
        ph = P_apply(p)
        v = A_apply(ph)
        den = rh @ v
        if den == 0.0:
            rep.breakdown = True
            break
        alpha = rho / den
        s = r - alpha * v
        rep.n_it += 1
        sn = np.linalg.norm(s)
        if sn / bn <= tol:
            x = x + alpha * ph
            rep.relres_history.append(sn / bn)
            rep.converged = True
            break
        sh = P_apply(s)
        t = A_apply(sh)
        tt = t @ t
        if tt == 0.0:
            rep.breakdown = True
            break
        omega = (t @ s) / tt
        x = x + alpha * ph + omega * sh
        r = s - omega * t
        rr = np.linalg.norm(r) / bn
        rep.relres_history.append(rr)
        if rr <= tol:
            rep.converged = True
            break
        if omega == 0.0:
            rep.breakdown = True
            break
    if not rep.relres_history:
        rep.relres_history.append(np.linalg.norm(r) / bn)
    rep.final_relres = np.linalg.norm(b - A_apply(x)) / bn
    return x, rep


def gmres(A_apply, P_apply, b, tol=1e-8, restart=50, max_it=2000):
    """Right-preconditioned restarted GMRES(m) (Saad), SURVEY.md §8(c).

    Conventions follow hx/krylov.py: x0 = 0, relres = ||r||/||b||, zero b ->
    converged at 0, tol > 0 validated, one A*P product = one iteration, the
    final true residual recomputed.  Arnoldi with modified Gram-Schmidt and
    Givens rotations; x <- x + P(V y) at every restart and on convergence.
    Convergence is declared on the TRUE residual of the updated iterate; if
    the Arnoldi estimate reached tol but the true residual did not, the
    method restarts from the true residual.
    """
    if tol <= 0:
        raise ValueError("tol must be positive")
    if restart < 1:
        raise ValueError("restart must be >= 1")
    P_apply = P_apply or (lambda v: v)
    b = np.asarray(b, float)
    n = b.size
    rep = Report()
    bn = np.linalg.norm(b)
    if bn == 0.0:
        rep.converged, rep.final_relres = True, 0.0
        rep.relres_history.append(0.0)
        return np.zeros(n), rep
    x = np.zeros(n)
    r = b.copy()
    beta = bn
    m = restart
    while rep.n_it < max_it:
        V = np.zeros((m + 1, n))
        Hh = np.zeros((m + 1, m))
        cs, sn = np.zeros(m), np.zeros(m)
        g = np.zeros(m + 1)
        g[0] = beta
        V[0] = r / beta
        k = 0
        happy = False
        for j in range(m):
            w = A_apply(P_apply(V[j]))
            rep.n_it += 1
            for i in range(j + 1):
                h = w @ V[i]
                Hh[i, j] = h
                w = w - h * V[i]
            hn = np.linalg.norm(w)
            Hh[j + 1, j] = hn
            for i in range(j):
                a, c = Hh[i, j], Hh[i + 1, j]
                Hh[i, j] = cs[i] * a + sn[i] * c
                Hh[i + 1, j] = -sn[i] * a + cs[i] * c
            den = math.hypot(Hh[j, j], Hh[j + 1, j])
            if den == 0.0:
                cs[j], sn[j] = 1.0, 0.0
            else:
                cs[j], sn[j] = Hh[j, j] / den, Hh[j + 1, j] / den
            Hh[j, j] = den
            Hh[j + 1, j] = 0.0
            g[j + 1] = -sn[j] * g[j]
            g[j] = cs[j] * g[j]
            est = abs(g[j + 1]) / bn
            rep.relres_history.append(est)
            k = j + 1
            if hn == 0.0:
                happy = True
                break
            V[j + 1] = w / hn
            if est <= tol or rep.n_it >= max_it:
                break
        y = scipy.linalg.solve_triangular(Hh[:k, :k], g[:k])
        x = x + P_apply(V[:k].T @ y)
        r = b - A_apply(x)
        beta = np.linalg.norm(r)
        if beta / bn <= tol:
            rep.converged = True
            break
        if happy or beta == 0.0:
            rep.breakdown = True
            break
    rep.final_relres = np.linalg.norm(b - A_apply(x)) / bn
    return x, rep


# ---------------------------------------------------------------------------
# Transient-loop pieces after the solve: flux recovery,
# CFL numbers, mass-balance residuals, pressure-driven step control.

def face_pressures(n_faces, free_faces, dirichlet_faces, dirichlet_values, pi_reduced):
    """Full per-face pressures with prescribed values inserted (hx/assembly.py:178-183)."""
    out = np.empty(n_faces)
    out[free_faces] = pi_reduced
    out[dirichlet_faces] = dirichlet_values
    return out


def recover_face_fluxes(e2f, f2e, floc, Binv, row_sums, diag, pi_full, p):
    """Per-face flux, positive out of the owner: interior faces the strong
    two-sided expression, hull faces the owner's one-sided flux
    (hx/assembly.py:334-356)."""
    pi_local = pi_full[e2f]
    q_one = row_sums * p[:, None] - np.einsum("eij,ej->ei", Binv, pi_local)
    lam = q_one + diag * pi_local
    owner, nbr = f2e[:, 0], f2e[:, 1]
    lo, ln = floc[:, 0], floc[:, 1]
    q = q_one[owner, lo].copy()
    it = np.flatnonzero(nbr >= 0)
    d_o = diag[owner[it], lo[it]]
    d_n = diag[nbr[it], ln[it]]
    q[it] = (d_n * lam[owner[it], lo[it]] - d_o * lam[nbr[it], ln[it]]) / (d_o + d_n)
    return q


def element_outflows(e2f, f2e, q):
    """Signed flux out of each element through its faces (hx/assembly.py:359-363)."""
    sign = np.where(f2e[e2f, 0] == np.arange(e2f.shape[0])[:, None], 1.0, -1.0)
    return sign * q[e2f]


def cfl(e2f, f2e, q, elem_volume, porosity, dt):
    """chi = outflow rate * dt / pore volume per element (hx/driver.py:67-71)."""
    out = element_outflows(e2f, f2e, q)
    rate = np.where(out > 0, out, 0.0).sum(axis=1)
    return rate * dt / (elem_volume * porosity)


def balance_residuals(e2f, f2e, q, elem_volume, accumulation, dt, p, p_prev=None, source=None):
    """Relative per-cell mass-balance residual (hx/assembly.py:367-387)."""
    signed = element_outflows(e2f, f2e, q)
    net = signed.sum(axis=1)
    gross = np.abs(signed).sum(axis=1)
    src = np.zeros(e2f.shape[0]) if source is None else elem_volume * source
    if math.isinf(dt):
        acc = np.zeros(e2f.shape[0])
    else:
        acc = accumulation * (p - (np.zeros(e2f.shape[0]) if p_prev is None else p_prev)) / dt
    scale = np.maximum(gross + np.abs(acc) + np.abs(src), np.abs(q).max() + 1e-300)
    return np.abs(acc + net - src) / scale


def next_dt(dt, dt_max, dt_mult, dp_target, dp_max):
    """Pressure-change driven step (hx/driver.py:50-53)."""
    ratio = dt_mult if dp_max <= 0 else min(dt_mult, dp_target / dp_max)
    return min(dt * ratio, dt_max)
