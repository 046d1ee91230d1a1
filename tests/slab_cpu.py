"""CPU stand-in for one slab of the partitioned solver -- TEST INFRASTRUCTURE.

It exposes the same part interface as ``parallel.CudaSlab`` with every
operation done by the oracle / scipy on torch CPU tensors, so the multi-rank
driver (``parallel.slab_gmres``, ``HaloExchange``, ``TorchComm``) can be
exercised with the gloo backend on CPU.  The product path never uses it.
"""

from __future__ import annotations

import math

import numpy as np
import scipy.sparse as sp
import torch

from oracle import edfa_oracle as O


def ext_sets(layout, global_sets):
    """Global restriction sets of the extended cells in ext face numbering
    (faces outside the extended box dropped)."""
    pos = np.full(int(max(layout.ext_faces.max(), max((s.max() for s in global_sets if s.size), default=0))) + 1,
                  -1, dtype=np.int64)
    pos[layout.ext_faces] = np.arange(layout.ext_faces.size)
    out = []
    for c in layout.ext_cells:
        s = np.asarray(global_sets[c], dtype=np.int64)
        m = pos[s]
        out.append(np.sort(m[m >= 0]))
    return out


def ext_stage1(layout, global_sets=None, dynamic=None):
    e = layout.blocks["ext"]
    if dynamic is not None:
        return O.build_stage1(e["A_ff"], e["A_fc"], e["A_cf"], dynamic=dynamic, no_fill=True)
    return O.build_stage1(e["A_ff"], e["A_fc"], e["A_cf"], sets=ext_sets(layout, global_sets), no_fill=True)


class CpuSlab:
    def __init__(self, layout, global_sets=None, dynamic=None):
        self.layout = lay = layout
        b = lay.blocks
        s1 = ext_stage1(lay, global_sets, dynamic)
        own = b["own_cells_in_ext"]
        H = s1.H.tocsr()[own][:, own]
        self.S_own = O.canonical(b["A_cc_own"] - H)
        self.ilu = O.ilu(self.S_own, 0.0, no_fill=True)
        self.ic = O.ic(-b["A_ff_own"], 0.0, no_fill=True)
        self.A_loc, self.A_cf_loc, self.A_fc_loc = b["A_loc"], b["A_cf_loc"], b["A_fc_loc"]
        nfo, nco = lay.n_faces, lay.n_cells
        nhf, nhc = lay.halo_faces.size, lay.halo_cells.size
        self.zext = torch.zeros(nfo + nco + nhf + nhc, dtype=torch.float64)
        self.tf_ext = torch.zeros(nfo + nhf, dtype=torch.float64)
        self.yc_ext = torch.zeros(nco + nhc, dtype=torch.float64)
        self.rhs = torch.from_numpy(b["rhs"].copy())

    def empty(self, *shape):
        return torch.empty(*shape, dtype=torch.float64)

    def gather(self, src, kind, q):
        idx = self.layout.send_faces[q] if kind == "f" else self.layout.send_cells[q]
        return src[torch.from_numpy(idx)].clone()

    def multidot(self, V, nvec, w, out):
        out[:nvec] = torch.from_numpy(V[:nvec].numpy() @ w.numpy())

    def multiaxpy(self, V, nvec, h, w_in, out, norm2):
        acc = h[:nvec].numpy() @ V[:nvec].numpy()
        o = acc if w_in is None else w_in.numpy() - acc
        out.copy_(torch.from_numpy(o))
        if norm2 is not None:
            norm2[0] = float(o @ o)

    def sync(self):   # CPU arithmetic has no deferred solve errors
        pass

    def axpby(self, a, x, b, y):
        y.copy_(a * x if b == 0.0 else a * x + b * y)

    # DCGS2 building blocks: numpy restatement of krylov.cu's k_dots2 /
    # dcgs2_coeffs_block / k_axpy2 (the coefficient algebra is the product's)
    def dcgs2_dots(self, V, j, out):
        Vn = V.numpy()
        out.zero_()
        out[:j + 1] = torch.from_numpy(Vn[:j + 1] @ Vn[j])
        out[64:65 + j] = torch.from_numpy(Vn[:j + 1] @ Vn[j + 1])

    def dcgs2_coeffs(self, j, m, dots, H, h1, coef, hcol):
        d = dots.numpy()
        Hn = H.numpy()            # (m, m+1): row i = Hessenberg column i
        if j == 0:
            h1[0] = d[64]
            coef[128], coef[129], coef[130] = 1.0, 1.0, -d[64]
            return
        a = d[:j].copy()
        aa, ab = a @ a, a @ d[64:64 + j]
        nu2 = d[j] - aa
        nu = math.sqrt(nu2) if nu2 > 0.0 else 0.0
        colv = h1.numpy()[:j] + a
        Hn[j - 1, :j] = colv
        Hn[j - 1, j] = nu
        hcol[:j] = torch.from_numpy(colv)
        hcol[j] = nu
        if nu == 0.0:
            coef.zero_()
            return
        inv = 1.0 / nu
        t = np.array([sum(Hn[i, r] * a[i] for i in range(max(0, r - 1), j)) for r in range(j + 1)])
        c = np.empty(j + 1)
        c[:j] = (d[64:64 + j] - t[:j]) * inv
        c[j] = ((d[64 + j] - ab) * inv - t[j]) * inv
        dd = t * inv + c
        h1[:j + 1] = torch.from_numpy(c)
        coef[:j] = torch.from_numpy(a * inv)
        coef[64:64 + j] = torch.from_numpy(dd[:j] - dd[j] * a * inv)
        coef[128], coef[129], coef[130] = inv, inv, -dd[j] * inv

    def dcgs2_update(self, V, j, coef):
        Vn, cf = V.numpy(), coef.numpy()
        u, w = Vn[j].copy(), Vn[j + 1].copy()
        q = cf[128] * u - cf[:j] @ Vn[:j]
        wt = cf[129] * w + cf[130] * u - cf[64:64 + j] @ Vn[:j]
        if j > 0:
            Vn[j] = q
        Vn[j + 1] = wt

    def fetch(self, t):
        a = t.numpy().copy()
        return lambda: a

    def copy(self, src, dst):
        dst.copy_(src)

    def spmv_ext(self, y):
        y.copy_(torch.from_numpy(self.A_loc @ self.zext.numpy()))

    def spmv_interior(self, y):
        from paper_2009_13916_b200.parallel import split_boundary_rows
        if not hasattr(self, "_split"):
            self._split = split_boundary_rows(self.A_loc, self.layout.n_own)
        y.copy_(torch.from_numpy(self._split[0] @ self.zext.numpy()))

    def spmv_boundary(self, y):
        _, rows, A_b = self._split
        if rows.size:
            y[torch.from_numpy(rows)] = torch.from_numpy(A_b @ self.zext.numpy())

    def apply_faces(self, r):
        nfo = self.layout.n_faces
        self.tf_ext[:nfo] = torch.from_numpy(-self.ic.apply(r[:nfo].numpy()))

    def apply_cells(self, r):
        nfo, nco = self.layout.n_faces, self.layout.n_cells
        u = r[nfo:nfo + nco].numpy() - self.A_cf_loc @ self.tf_ext.numpy()
        self.yc_ext[:nco] = torch.from_numpy(self.ilu.apply(u))

    def apply_finish(self, y):
        nfo, nco = self.layout.n_faces, self.layout.n_cells
        a = self.A_fc_loc @ self.yc_ext.numpy()
        y[:nfo] = torch.from_numpy(self.tf_ext[:nfo].numpy() + self.ic.apply(a))
        y[nfo:nfo + nco] = self.yc_ext[:nco]


def block_jacobi_reference(system, layouts, global_sets=None, dynamic=None, tol=1e-8, restart=50):
    """The oracle's EDFA with slab-block-diagonal inner factors (what the
    partitioned solver computes), solved with the oracle's GMRES."""
    A_ff, A_fc, A_cf, A_cc = (sp.csr_matrix(getattr(system, n)) for n in ("A_ff", "A_fc", "A_cf", "A_cc"))
    if dynamic is not None:
        s1 = O.build_stage1(A_ff, A_fc, A_cf, dynamic=dynamic, no_fill=True)
    else:
        s1 = O.build_stage1(A_ff, A_fc, A_cf, sets=global_sets, no_fill=True)
    fpart = np.empty(A_ff.shape[0], dtype=np.int64)
    cpart = np.empty(A_cc.shape[0], dtype=np.int64)
    for lay in layouts:
        fpart[lay.own_faces] = lay.rank
        cpart[lay.own_cells] = lay.rank

    def mask(M, p):
        M = sp.coo_matrix(M)
        keep = p[M.row] == p[M.col]
        return O.canonical(sp.coo_matrix((M.data[keep], (M.row[keep], M.col[keep])), shape=M.shape))

    S_bj = mask(O.canonical(A_cc - s1.H), cpart)
    ilu = O.ilu(S_bj, 0.0, no_fill=True)
    ic = O.ic(-mask(A_ff, fpart), 0.0, no_fill=True)
    nf = A_ff.shape[0]

    def P(r):
        t_f = -ic.apply(r[:nf])
        t_c = ilu.apply(r[nf:] - A_cf @ t_f)
        return np.concatenate([t_f + ic.apply(A_fc @ t_c), t_c])

    A = system.full_matrix()
    x, rep = O.gmres(lambda v: A @ v, P, system.rhs(), tol=tol, restart=restart)
    return x, rep, S_bj
