"""Vectorised RT0 mixed-hybrid / FV assembly of the 2x2 block system.

Input producer for the EDFA path (done on the host
in numpy so BASELINE configs 2-5 can be generated on the GPU box).  It
restates hx/assembly.py without its per-cell Python loop (hx/assembly.py:
252-274):

* elemental ``B^E`` by 2x2x2 Gauss + contravariant Piola   (57-73)
* ``Binv`` cleaned of relative dust < 1e-13 and re-symmetrised (76-88)
* A_ff = -sum_E P_E Binv^E P_E^T, A_fc from Binv row sums   (208-227)
* balance rows with the strong two-sided flux on interior faces (232-276)
* Dirichlet elimination into the RHS                        (283-299)
* ``update_accumulation`` for backward-Euler steps          (314-333)

Blocks come out as canonical scipy CSR (sorted, duplicate-free, no stored
zeros), exactly the storage convention of hx/sparse.py:28-34.
"""

from __future__ import annotations

import dataclasses
import math
from dataclasses import dataclass

import numpy as np
import scipy.sparse as sp

from .mesh import (Boundaries, Conductivity, HexGrid, RockProps, gauss3,
                   rt0_reference, shape_grad)

_BINV_CLEAN = 1e-13


def canonical(A) -> sp.csr_matrix:
    """Sorted, duplicate-summed CSR without explicit zeros (hx/sparse.py:28-34)."""
    A = sp.csr_matrix(A)
    A.sum_duplicates()
    A.sort_indices()
    A.eliminate_zeros()
    return A


@dataclass(frozen=True)
class ElementOps:
    Binv: np.ndarray       # (n, 6, 6)
    row_sums: np.ndarray   # (n, 6)
    diag: np.ndarray       # (n, 6)


def element_ops(grid: HexGrid, field: Conductivity, gamma: float) -> ElementOps:
    Kinv = np.linalg.inv(field.tensors)
    Kinv = 0.5 * (Kinv + Kinv.transpose(0, 2, 1))
    xyz = grid.elem_coords()
    pts, wts = gauss3()
    B = np.zeros((xyz.shape[0], 6, 6))
    for p, w in zip(pts, wts):
        J = np.matmul(xyz.transpose(0, 2, 1), shape_grad(p))          # (e, 3, 3)
        det = np.linalg.det(J)
        if np.any(det <= 0):
            raise ValueError("non-positive Jacobian")
        M = np.matmul(J, rt0_reference(p).T)                          # (e, 3, 6)
        B += np.matmul(M.transpose(0, 2, 1), np.matmul(Kinv, M)) * (w / det)[:, None, None]
    B *= gamma
    B = 0.5 * (B + B.transpose(0, 2, 1))
    Bi = np.linalg.inv(B)
    Bi = 0.5 * (Bi + Bi.transpose(0, 2, 1))
    scale = np.abs(Bi).max(axis=2, keepdims=True)
    Bi[np.abs(Bi) < _BINV_CLEAN * scale] = 0.0
    Bi = 0.5 * (Bi + Bi.transpose(0, 2, 1))
    return ElementOps(Bi, Bi.sum(axis=2), Bi[:, np.arange(6), np.arange(6)].copy())


@dataclass(frozen=True)
class BlockSystem:
    """Assembled blocks in reduced (free-face) numbering; field names match
    hx/assembly.py:135-183 so either container can be handed to the EDFA
    drop-in."""

    A_ff: sp.csr_matrix
    A_fc: sp.csr_matrix
    A_cf: sp.csr_matrix
    A_cc: sp.csr_matrix
    rhs_f: np.ndarray
    rhs_c: np.ndarray
    dt: float
    free_faces: np.ndarray
    face_index: np.ndarray
    dirichlet_faces: np.ndarray
    dirichlet_values: np.ndarray
    A_cc_steady: sp.csr_matrix
    accumulation: np.ndarray
    rhs_c_base: np.ndarray
    ops: ElementOps
    grid: HexGrid

    @property
    def n_free_faces(self) -> int:
        return self.free_faces.size

    @property
    def n_cells(self) -> int:
        return self.A_cc.shape[0]

    @property
    def n_unknowns(self) -> int:
        return self.n_free_faces + self.n_cells

    def full_matrix(self) -> sp.csr_matrix:
        return canonical(sp.bmat([[self.A_ff, self.A_fc],
                                  [self.A_cf, self.A_cc]], format="csr"))

    def rhs(self) -> np.ndarray:
        return np.concatenate([self.rhs_f, self.rhs_c])

    def split(self, u):
        return u[:self.n_free_faces], u[self.n_free_faces:]


def assemble(grid: HexGrid, field: Conductivity, props: RockProps,
             bc: Boundaries, dt: float, p_prev=None) -> BlockSystem:
    """Block system for one step (``dt=math.inf``: steady)."""
    if not dt > 0:
        raise ValueError("dt must be positive (math.inf for steady state)")
    n_e, n_f = grid.n_elems, grid.n_faces
    dfaces, dvals, nfaces, nvals = bc.resolve(grid)
    if math.isinf(dt) and dfaces.size == 0:
        raise ValueError("steady problem without a prescribed pressure is singular")
    ops = element_ops(grid, field, props.gamma)
    Bi, rs, dg = ops.Binv, ops.row_sums, ops.diag
    e2f = grid.elem_to_faces
    cells = np.arange(n_e)

    # flux-continuity rows
    r = np.repeat(e2f, 6, axis=1).ravel()
    c = np.tile(e2f, (1, 6)).ravel()
    A_ff_full = sp.coo_matrix((-Bi.reshape(n_e, 36).ravel(), (r, c)),
                              shape=(n_f, n_f)).tocsr()
    A_fc_full = sp.coo_matrix((rs.ravel(), (e2f.ravel(), np.repeat(cells, 6))),
                              shape=(n_f, n_e)).tocsr()
    f_pi = np.zeros(n_f)
    if nfaces.size:
        f_pi[nfaces] = nvals * grid.face_area[nfaces]

    # balance rows with the strong flux (interior) / one-sided flux (hull)
    nb = grid.neighbors()                                     # (n, 6)
    inner = nb >= 0
    fe = grid.face_to_elems[e2f]
    own = fe[:, :, 0] == cells[:, None]
    nloc = np.where(own, grid.face_local[e2f, 1], grid.face_local[e2f, 0])
    nloc = np.where(inner, nloc, -1)
    d_oth = np.zeros((n_e, 6))
    d_oth[inner] = dg[nb[inner], nloc[inner]]
    w = np.where(inner, d_oth / np.where(inner, dg + d_oth, 1.0), 1.0)

    coef = -np.einsum("ei,eij->ej", w, Bi)
    coef = np.where(inner, coef + w * dg, coef)
    cf_r = [np.repeat(cells, 6)]
    cf_c = [e2f.ravel()]
    cf_v = [coef.ravel()]
    cc_r = [cells]
    cc_c = [cells]
    cc_v = [np.einsum("ei,ei->e", w, rs)]
    for slot in range(6):
        m = np.flatnonzero(inner[:, slot])
        if m.size == 0:
            continue
        nbr, ln = nb[m, slot], nloc[m, slot]
        wf = 1.0 - w[m, slot]
        far = wf[:, None] * Bi[nbr, ln, :]                      # (k, 6)
        far[np.arange(m.size), ln] = 0.0
        cf_r.append(np.repeat(m, 6))
        cf_c.append(e2f[nbr].ravel())
        cf_v.append(far.ravel())
        cc_r.append(m)
        cc_c.append(nbr)
        cc_v.append(-wf * rs[nbr, ln])
    A_cf_full = sp.coo_matrix((np.concatenate(cf_v),
                               (np.concatenate(cf_r), np.concatenate(cf_c))),
                              shape=(n_e, n_f)).tocsr()
    A_cc = canonical(sp.coo_matrix((np.concatenate(cc_v),
                                    (np.concatenate(cc_r), np.concatenate(cc_c))),
                                   shape=(n_e, n_e)))

    keep = np.ones(n_f, bool)
    keep[dfaces] = False
    free = np.flatnonzero(keep)
    fidx = np.full(n_f, -1, np.int64)
    fidx[free] = np.arange(free.size)
    A_ff_rows = A_ff_full[free]
    rhs_f = f_pi[free]
    rhs_c = np.zeros(n_e)
    if dfaces.size:
        rhs_f = rhs_f - A_ff_rows[:, dfaces] @ dvals
        rhs_c = rhs_c - A_cf_full[:, dfaces] @ dvals
    sysm = BlockSystem(
        A_ff=canonical(A_ff_rows[:, free]), A_fc=canonical(A_fc_full[free]),
        A_cf=canonical(A_cf_full[:, free]), A_cc=A_cc, rhs_f=rhs_f,
        rhs_c=rhs_c, dt=math.inf, free_faces=free, face_index=fidx,
        dirichlet_faces=dfaces, dirichlet_values=dvals, A_cc_steady=A_cc,
        accumulation=grid.elem_volume * props.storage(n_e), rhs_c_base=rhs_c,
        ops=ops, grid=grid)
    if math.isinf(dt):
        return sysm
    return update_accumulation(sysm, dt, p_prev)


def update_accumulation(system, dt: float, p_prev=None):
    """New system for step ``dt``: only A_cc and rhs_c change; the face
    blocks are shared by identity (hx/assembly.py:314-333)."""
    if not dt > 0:
        raise ValueError("dt must be positive (math.inf for steady state)")
    if math.isinf(dt):
        return dataclasses.replace(system, dt=dt, A_cc=system.A_cc_steady,
                                   rhs_c=system.rhs_c_base)
    n = system.n_cells
    p_prev = np.zeros(n) if p_prev is None else np.asarray(p_prev, float)
    A_cc = canonical(system.A_cc_steady
                     + sp.diags(system.accumulation / dt, format="csr"))
    rhs_c = system.rhs_c_base + system.accumulation * p_prev / dt
    return dataclasses.replace(system, dt=dt, A_cc=A_cc, rhs_c=rhs_c)
