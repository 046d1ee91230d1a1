"""Z-slab partitioned EDFA + GMRES(m) over several GPUs.

Partitioning (hx/grid.py:49-50, 100-129): cells are numbered i + nx(j + ny k)
and every face family is k-slowest, so a slab of cell layers [k0, k1) is one
contiguous cell range; a face belongs to the slab of its owner cell (the
lower-indexed cell, ``face_to_elems[f, 0]``).  A rank keeps the rows of its
own faces and cells; the local vector is ``[own faces | own cells]``.

* Setup.  Stage-1 rows (restricted solves, G~, F~, H~) are independent per
  cell.  Each rank computes them on its *extended* subsystem --
  the slab plus ``halo`` cell layers on each side, a read-only copy of the
  neighbours' rows -- so the rows of its own cells are exactly the global
  ones.  It keeps the block-Jacobi inner factors
      IC(0) of -A_ff[own, own],    ILU(0) of S~[own, own] = A_cc - H~ on own x own,
  so no triangular solve crosses a slab boundary.
* Apply (hx/precond.py:311-320) and SpMV exchange one layer of halo values
  (faces for ``A_cf``, cells for ``A_fc``); Krylov dot products are summed
  over ranks (NCCL allreduce over NVLink on the GPU path).

The driver is written over *parts*: a process holds one part per GPU in
production (``torch.distributed`` over NCCL), or several parts on one device
when emulating k slabs (the halo copies are then local).  Nothing here
computes on the host: parts do their arithmetic through libedfa.
"""

from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field

import numpy as np
import scipy.sparse as sp
import torch

from . import _lib as L
from .krylov import SolveReport

# ---------------------------------------------------------------------------
# host partition (integer bookkeeping only)

PATTERN_REACH = {"base": 0, "A": 2, "B": 3, "C": 1, "D": 2, "E": 1}


def halo_layers(kind: str, prototype: str = "A", dynamic=None) -> int:
    """Cell layers of read-only halo that make the own rows of G~, F~ and
    H~[own, own] exact: the pattern's reach in cells plus one (the faces of
    a pattern need both of their cells for a complete A_ff row)."""
    if dynamic is not None or kind == "dynamic":
        n_ent = dynamic.n_ent if dynamic is not None else 4
        return 2 + n_ent
    if kind == "base":
        return 1
    return PATTERN_REACH[prototype] + 1


def slab_bounds(nz: int, parts: int):
    if parts < 1 or parts > nz:
        raise ValueError(f"cannot cut {nz} cell layers into {parts} slabs")
    return [(r * nz // parts, (r + 1) * nz // parts) for r in range(parts)]


def _canon(A):
    A = sp.csr_matrix(A)
    A.sum_duplicates()
    A.sort_indices()
    return A


@dataclass
class SlabLayout:
    """Rows, halo lists and local blocks of one slab (all numpy / scipy)."""

    rank: int
    size: int
    k0: int
    k1: int
    e0: int
    e1: int
    nxyz: tuple
    own_faces: np.ndarray          # free-face ids, sorted
    own_cells: np.ndarray          # cell ids, contiguous
    halo_faces: np.ndarray         # ordered by (owner rank, id)
    halo_cells: np.ndarray
    recv_faces: dict               # peer -> (start, stop) into halo_faces
    recv_cells: dict
    send_faces: dict = field(default_factory=dict)   # peer -> positions into own_faces
    send_cells: dict = field(default_factory=dict)
    ext_faces: np.ndarray = None
    ext_cells: np.ndarray = None
    blocks: dict = field(default_factory=dict)

    @property
    def n_faces(self) -> int:
        return self.own_faces.size

    @property
    def n_cells(self) -> int:
        return self.own_cells.size

    @property
    def n_own(self) -> int:
        return self.n_faces + self.n_cells


def _ordered_halo(ids, owner):
    order = np.lexsort((ids, owner))
    ids, owner = ids[order], owner[order]
    recv = {}
    for q in np.unique(owner):
        w = np.flatnonzero(owner == q)
        recv[int(q)] = (int(w[0]), int(w[-1]) + 1)
    return ids, owner, recv


def build_layouts(system, parts: int, halo: int, ranks=None):
    """Slab layouts of a BlockSystem on an nx*ny*nz box (hexflow numbering).

    ``ranks`` limits the (expensive) local block extraction to the listed
    slabs; the halo lists of every slab are always computed (they define
    what each slab sends)."""
    grid = system.grid
    nx, ny, nz = grid.nx, grid.ny, grid.nz
    nxy = nx * ny
    nf = system.n_free_faces
    bounds = slab_bounds(nz, parts)
    layer_part = np.empty(nz, dtype=np.int64)
    for r, (a, b) in enumerate(bounds):
        layer_part[a:b] = r
    f2e = np.asarray(grid.face_to_elems)
    free = np.asarray(system.free_faces)
    face_part = layer_part[f2e[free, 0] // nxy]
    cell_part = layer_part[np.arange(system.n_cells) // nxy]
    A = _canon(system.full_matrix())
    ranks = range(parts) if ranks is None else ranks
    lays = []
    for r, (k0, k1) in enumerate(bounds):
        own_f = np.flatnonzero(face_part == r)
        own_c = np.arange(k0 * nxy, k1 * nxy)
        rows = np.concatenate([own_f, nf + own_c])
        Ar = A[rows]
        cols = np.unique(Ar.indices)
        hf = cols[(cols < nf)]
        hf = hf[face_part[hf] != r]
        hc = cols[cols >= nf] - nf
        hc = hc[cell_part[hc] != r]
        hf, hf_own, recv_f = _ordered_halo(hf, face_part[hf])
        hc, hc_own, recv_c = _ordered_halo(hc, cell_part[hc])
        e0, e1 = max(0, k0 - halo), min(nz, k1 + halo)
        lay = SlabLayout(r, parts, k0, k1, e0, e1, (nx, ny, nz), own_f, own_c, hf, hc, recv_f, recv_c)
        if r in ranks:
            _local_blocks(system, A, lay, nf, f2e, free, nxy)
        lays.append(lay)
    for q, lq in enumerate(lays):          # what slab q receives, slab r sends
        for r, (a, b) in lq.recv_faces.items():
            lays[r].send_faces[q] = np.searchsorted(lays[r].own_faces, lq.halo_faces[a:b])
        for r, (a, b) in lq.recv_cells.items():
            lays[r].send_cells[q] = np.searchsorted(lays[r].own_cells, lq.halo_cells[a:b])
    return lays


def _local_blocks(system, A, lay, nf, f2e, free, nxy):
    """Local rows with local column numbering and the extended subsystem."""
    nfo, nco = lay.n_faces, lay.n_cells
    nhf, nhc = lay.halo_faces.size, lay.halo_cells.size
    n_all = nf + system.n_cells
    cmap = np.full(n_all, -1, dtype=np.int64)
    cmap[lay.own_faces] = np.arange(nfo)
    cmap[nf + lay.own_cells] = nfo + np.arange(nco)
    cmap[lay.halo_faces] = nfo + nco + np.arange(nhf)
    cmap[nf + lay.halo_cells] = nfo + nco + nhf + np.arange(nhc)
    rows = np.concatenate([lay.own_faces, nf + lay.own_cells])

    def remap(M, rows, cmap, n_cols):
        M = M[rows]
        c = cmap[M.indices]
        if (c < 0).any():
            raise AssertionError("halo lists miss a column of the local rows")
        return _canon(sp.csr_matrix((M.data, c, M.indptr), shape=(M.shape[0], n_cols)))

    b = lay.blocks
    b["A_loc"] = remap(A, rows, cmap, nfo + nco + nhf + nhc)
    fmap = np.full(nf, -1, dtype=np.int64)
    fmap[lay.own_faces] = np.arange(nfo)
    fmap[lay.halo_faces] = nfo + np.arange(nhf)
    cmap_c = np.full(system.n_cells, -1, dtype=np.int64)
    cmap_c[lay.own_cells] = np.arange(nco)
    cmap_c[lay.halo_cells] = nco + np.arange(nhc)
    b["A_cf_loc"] = remap(system.A_cf.tocsr(), lay.own_cells, fmap, nfo + nhf)
    b["A_fc_loc"] = remap(system.A_fc.tocsr(), lay.own_faces, cmap_c, nco + nhc)
    b["A_ff_own"] = _canon(system.A_ff.tocsr()[lay.own_faces][:, lay.own_faces])
    b["A_cc_own"] = _canon(system.A_cc.tocsr()[lay.own_cells][:, lay.own_cells])
    # extended subsystem: cells of layers [e0, e1) and every free face of theirs
    ext_c = np.arange(lay.e0 * nxy, lay.e1 * nxy)
    lay.ext_cells = ext_c
    lo, hi = lay.e0 * nxy, lay.e1 * nxy
    fe = f2e[free]
    in_ext = ((fe[:, 0] >= lo) & (fe[:, 0] < hi)) | ((fe[:, 1] >= lo) & (fe[:, 1] < hi))
    ext_f = np.flatnonzero(in_ext)
    lay.ext_faces = ext_f
    b["ext"] = {
        "A_ff": _canon(system.A_ff.tocsr()[ext_f][:, ext_f]),
        "A_fc": _canon(system.A_fc.tocsr()[ext_f][:, ext_c]),
        "A_cf": _canon(system.A_cf.tocsr()[ext_c][:, ext_f]),
        "A_cc": _canon(system.A_cc.tocsr()[ext_c][:, ext_c]),
    }
    b["own_cells_in_ext"] = lay.own_cells - lo
    b["own_faces_in_ext"] = np.searchsorted(ext_f, lay.own_faces)
    # topology of the extended box for the static-pattern kernel: ext cells'
    # faces in a compact numbering, neighbours outside the box cut off
    grid = system.grid
    e2f = np.asarray(grid.elem_to_faces)[ext_c]
    all_f, inv = np.unique(e2f, return_inverse=True)
    e2f_loc = inv.reshape(e2f.shape)
    fe_all = f2e[all_f]
    nb = np.where(fe_all[inv.reshape(e2f.shape), 0] == ext_c[:, None],
                  fe_all[inv.reshape(e2f.shape), 1], fe_all[inv.reshape(e2f.shape), 0])
    nb = np.where((nb >= lo) & (nb < hi), nb - lo, -1)
    fi = np.asarray(system.face_index)[all_f]
    ext_pos = np.full(nf, -1, dtype=np.int64)
    ext_pos[ext_f] = np.arange(ext_f.size)
    fidx = np.where(fi >= 0, ext_pos[np.maximum(fi, 0)], -1)
    b["ext_topology"] = (e2f_loc.astype(np.int32), nb.astype(np.int32), fidx.astype(np.int32))
    b["rhs"] = np.concatenate([system.rhs_f[lay.own_faces], system.rhs_c[lay.own_cells]])


def _sub_face_keys(nx, ny, nz, s0, nzs):
    """Global face ids and owner cell layers of the faces of the sub-box of
    cell layers [s0, s0 + nzs) (hx/grid.py:97-129 numbering: families x, y, z,
    each k-slowest; a face is owned by its lower-indexed cell)."""
    nxf, nyf = (nx + 1) * ny * nzs, nx * (ny + 1) * nzs
    NXF, NYF = (nx + 1) * ny * nz, nx * (ny + 1) * nz
    f = np.arange(nxf)
    i, j, k = f % (nx + 1), (f // (nx + 1)) % ny, f // ((nx + 1) * ny)
    gx, lx = i + (nx + 1) * (j + ny * (k + s0)), k + s0
    f = np.arange(nyf)
    i, j, k = f % nx, (f // nx) % (ny + 1), f // (nx * (ny + 1))
    gy, ly = NXF + i + nx * (j + (ny + 1) * (k + s0)), k + s0
    f = np.arange(nx * ny * (nzs + 1))
    i, j, kp = f % nx, (f // nx) % ny, f // (nx * ny)
    gz, lz = NXF + NYF + i + nx * (j + ny * (kp + s0)), np.maximum(kp + s0 - 1, 0)
    return np.concatenate([gx, gy, gz]), np.concatenate([lx, ly, lz])


def build_slab_layout(sub, s0: int, nz: int, parts: int, rank: int, halo: int) -> SlabLayout:
    """The layout of slab ``rank`` built from its own sub-box only -- no
    global system on any process (host memory O(slab)).

    ``sub`` is the BlockSystem of the cell layers [s0, s1) with s0 = max(0,
    e0 - 1), s1 = min(nz, e1 + 1) around the extended slab [e0, e1) =
    [k0 - halo, k1 + halo) (configs.slab_case): every row whose cells lie in
    layers [s0 + 1, s1 - 2] equals the global row.  Entries are matched
    across ranks by global ids (cells i + nx(j + ny k), faces by
    _sub_face_keys); halo lists are ordered by (owner slab, global id), the
    order build_layouts uses, so the local blocks are the global ones."""
    grid = sub.grid
    nx, ny, nzs = grid.nx, grid.ny, grid.nz
    s1 = s0 + nzs
    nxy = nx * ny
    bounds = slab_bounds(nz, parts)
    k0, k1 = bounds[rank]
    e0, e1 = max(0, k0 - halo), min(nz, k1 + halo)
    if not (s0 <= max(e0 - 1, 0) and min(e1 + 1, nz) <= s1):
        raise ValueError("the sub-box does not cover the extended slab plus one layer")
    layer_part = np.empty(nz, dtype=np.int64)
    for r, (a, b) in enumerate(bounds):
        layer_part[a:b] = r
    free = np.asarray(sub.free_faces)
    nf = free.size
    gface, lface = _sub_face_keys(nx, ny, nz, s0, nzs)
    fkey, flay = gface[free], lface[free]
    face_part = layer_part[flay]
    n_c = sub.n_cells
    clay = np.arange(n_c) // nxy + s0
    ckey = np.arange(n_c) + s0 * nxy
    cell_part = layer_part[clay]
    A = _canon(sub.full_matrix())
    own_f = np.flatnonzero(face_part == rank)
    own_c = np.flatnonzero(cell_part == rank)
    rows = np.concatenate([own_f, nf + own_c])
    cols = np.unique(A[rows].indices)
    hf = cols[cols < nf]
    hf = hf[face_part[hf] != rank]
    hc = cols[cols >= nf] - nf
    hc = hc[cell_part[hc] != rank]

    def ordered(ids, owner, key):
        o = np.lexsort((key[ids], owner[ids]))
        ids = ids[o]
        recv = {}
        for q in np.unique(owner[ids]):
            w = np.flatnonzero(owner[ids] == q)
            recv[int(q)] = (int(w[0]), int(w[-1]) + 1)
        return ids, recv

    hf, recv_f = ordered(hf, face_part, fkey)
    hc, recv_c = ordered(hc, cell_part, ckey)
    lay = SlabLayout(rank, parts, k0 - s0, k1 - s0, e0 - s0, e1 - s0, (nx, ny, nzs), own_f, own_c, hf, hc,
                     recv_f, recv_c)
    lay.global_bounds = (k0, k1, e0, e1, s0, s1)
    lay.face_keys, lay.cell_keys = fkey, ckey
    # what each other slab needs from this one: this slab's entries among the
    # columns of that slab's complete rows in the sub-box (sorted by global id)
    lo = s0 + 1 if s0 > 0 else 0
    hi = s1 - 2 if s1 < nz else nz - 1
    complete_f = (flay >= lo) & (flay <= hi)
    complete_c = (clay >= lo) & (clay <= hi)
    for q in sorted(set(face_part[complete_f].tolist()) | set(cell_part[complete_c].tolist())):
        if q == rank:
            continue
        qrows = np.concatenate([np.flatnonzero(complete_f & (face_part == q)),
                                nf + np.flatnonzero(complete_c & (cell_part == q))])
        qc = np.unique(A[qrows].indices)
        sf = qc[(qc < nf)]
        sf = sf[face_part[sf] == rank]
        sc = qc[qc >= nf] - nf
        sc = sc[cell_part[sc] == rank]
        if sf.size:
            lay.send_faces[q] = np.searchsorted(own_f, sf[np.argsort(fkey[sf], kind="stable")])
        if sc.size:
            lay.send_cells[q] = np.searchsorted(own_c, sc[np.argsort(ckey[sc], kind="stable")])
    _local_blocks(sub, A, lay, nf, np.asarray(grid.face_to_elems), free, nxy)
    return lay


def split_boundary_rows(A_loc, n_own):
    """(interior, boundary rows, boundary block) of a slab's local matrix:
    interior = A_loc with the rows that reference halo columns emptied (it
    writes 0 there), boundary = those rows compacted.  The interior SpMV runs
    while the halo exchange is in flight; the boundary rows follow it."""
    A = sp.csr_matrix(A_loc)
    touches = np.zeros(A.shape[0], dtype=bool)
    if A.nnz:
        row_of = np.repeat(np.arange(A.shape[0]), np.diff(A.indptr))
        touches[row_of[A.indices >= n_own]] = True
    rows = np.flatnonzero(touches)
    keep = np.repeat(~touches, np.diff(A.indptr))
    A_int = sp.csr_matrix((A.data[keep], A.indices[keep],
                           np.concatenate([[0], np.cumsum(np.diff(A.indptr) * ~touches)])), shape=A.shape)
    return A_int, rows, A[rows]


def scatter_solution(layouts, xs, n_free_faces, n_cells):
    """Global solution from the per-slab local vectors (host)."""
    x = np.empty(n_free_faces + n_cells)
    for lay, xl in zip(layouts, xs):
        xl = xl.detach().cpu().numpy() if isinstance(xl, torch.Tensor) else np.asarray(xl)
        x[lay.own_faces] = xl[:lay.n_faces]
        x[n_free_faces + lay.own_cells] = xl[lay.n_faces:]
    return x


# ---------------------------------------------------------------------------
# communication

class LocalComm:
    """Single process: every part is local, reductions are local sums."""

    rank_of_part = None

    def __init__(self, parts: int):
        self.rank_of_part = [0] * parts
        self.rank = 0

    def allreduce_(self, t: torch.Tensor) -> None:
        return None

    def p2p(self, sends, recvs) -> None:
        if sends or recvs:
            raise RuntimeError("LocalComm has no remote peers")

    def p2p_start(self, sends, recvs):
        self.p2p(sends, recvs)
        return []

    @staticmethod
    def p2p_wait(works) -> None:
        return None


class TorchComm:
    """torch.distributed process group (NCCL on GPUs, gloo on CPU); one or
    more slabs per process, ``rank_of_part[s]`` = process holding slab s."""

    def __init__(self, rank_of_part, group=None):
        import torch.distributed as dist
        self.dist = dist
        self.group = group
        self.rank = dist.get_rank(group)
        self.rank_of_part = list(rank_of_part)

    def allreduce_(self, t: torch.Tensor) -> None:
        self.dist.all_reduce(t, group=self.group)

    def p2p_start(self, sends, recvs):
        """Issue the P2P operations (one NCCL group); returns the pending works."""
        d = self.dist
        ops = [d.P2POp(d.isend, t, peer, self.group) for peer, t in sends]
        ops += [d.P2POp(d.irecv, t, peer, self.group) for peer, t in recvs]
        return d.batch_isend_irecv(ops) if ops else []

    @staticmethod
    def p2p_wait(works) -> None:
        for req in works:        # stream-ordered: the compute stream waits for NCCL's
            req.wait()

    def p2p(self, sends, recvs) -> None:
        """sends/recvs: lists of (peer process, tensor); matched in order."""
        self.p2p_wait(self.p2p_start(sends, recvs))


class HaloExchange:
    """Moves own-entry values of each slab into its neighbours' halo slots."""

    def __init__(self, parts, comm):
        self.parts = parts                  # local parts (objects with .layout)
        self.comm = comm
        self.by_slab = {p.layout.rank: p for p in parts}

    def run(self, kind: str, src, dst) -> None:
        """kind 'f' or 'c'; src[i] own-entry vector, dst[i] halo vector of parts[i]."""
        self.run_many([(kind, src, dst)])

    def run_many(self, jobs) -> None:
        """Several exchanges [(kind, src, dst), ...] in ONE batch of P2P
        operations (one NCCL group launch instead of one per kind)."""
        self.comm.p2p_wait(self.start_many(jobs))

    def start_many(self, jobs):
        """run_many without the final wait: returns the pending works (local
        copies are done; the remote halves are in flight on NCCL's stream)."""
        rank_of = self.comm.rank_of_part
        remote_s, remote_r = [], []
        sends = {}
        for ji, (kind, src, dst) in enumerate(jobs):
            send_attr = "send_faces" if kind == "f" else "send_cells"
            recv_attr = "recv_faces" if kind == "f" else "recv_cells"
            bufs = {}
            for p, s in zip(self.parts, src):
                for q in sorted(getattr(p.layout, send_attr)):
                    bufs[(p.layout.rank, q)] = p.gather(s, kind, q)
            for p, d in zip(self.parts, dst):
                for q, (a, b) in sorted(getattr(p.layout, recv_attr).items()):
                    if q in self.by_slab:
                        d[a:b].copy_(bufs[(q, p.layout.rank)])
                    else:
                        remote_r.append(((p.layout.rank, q, ji), rank_of[q], d[a:b]))
            for (src_slab, q), buf in bufs.items():
                if q not in self.by_slab:
                    sends[(src_slab, q, ji)] = (rank_of[q], buf)
        if sends or remote_r:
            # matched in order on both ends of every process pair: sends sorted
            # by (source slab, target slab, job), receives by (local slab,
            # source slab, job) -- z-slabs of one process are contiguous, so a
            # process pair shares one slab boundary
            remote_s = [sends[k] for k in sorted(sends)]
            remote_r = [(peer, t) for _, peer, t in sorted(remote_r, key=lambda e: e[0])]
            return self.comm.p2p_start(remote_s, remote_r)
        return []


# ---------------------------------------------------------------------------
# device part

class CudaSlab:
    """One slab on the current CUDA device; every operation is a libedfa call."""

    def __init__(self, layout: SlabLayout, *, kind="static", prototype="A", dynamic=None,
                 tau_filt=0.0, filtration="none", face_drop_tol=0.0, schur_drop_tol=0.0, no_fill=True):
        from .device import DeviceCsr, DeviceSystem, ctx
        self.layout = layout
        self.opts = dict(kind=kind, prototype=prototype, dynamic=dynamic, tau_filt=tau_filt,
                         filtration=filtration, face_drop_tol=face_drop_tol, schur_drop_tol=schur_drop_tol,
                         no_fill=no_fill)
        self.lib = L.lib()
        self.ctx = ctx()
        b = layout.blocks
        dev = torch.device("cuda", torch.cuda.current_device())
        i32 = lambda a: torch.from_numpy(np.ascontiguousarray(a, dtype=np.int32)).to(dev)  # noqa: E731
        self.A_loc = DeviceCsr.from_scipy(b["A_loc"])
        A_int, brows, A_bnd = split_boundary_rows(b["A_loc"], layout.n_own)
        self.A_int, self.A_bnd = DeviceCsr.from_scipy(A_int), DeviceCsr.from_scipy(A_bnd)
        self.A_cf_loc = DeviceCsr.from_scipy(b["A_cf_loc"])
        self.A_fc_loc = DeviceCsr.from_scipy(b["A_fc_loc"])
        self.A_ff_own = DeviceCsr.from_scipy(b["A_ff_own"])
        self.A_cc_own = DeviceCsr.from_scipy(b["A_cc_own"])
        e = b["ext"]
        self.ext = DeviceSystem(*(DeviceCsr.from_scipy(e[n]) for n in ("A_ff", "A_fc", "A_cf", "A_cc")))
        self.ext.topology = tuple(i32(a) for a in b["ext_topology"])
        self.own_in_ext = i32(b["own_cells_in_ext"])
        cm = np.full(layout.ext_cells.size, -1, dtype=np.int32)
        cm[b["own_cells_in_ext"]] = np.arange(layout.n_cells, dtype=np.int32)
        self.cell_map = i32(cm)
        self.brows = i32(brows)
        self.send = {("f", q): i32(v) for q, v in layout.send_faces.items()}
        self.send.update({("c", q): i32(v) for q, v in layout.send_cells.items()})
        self.rhs = torch.from_numpy(b["rhs"]).to(dev)
        nfo, nco = layout.n_faces, layout.n_cells
        nhf, nhc = layout.halo_faces.size, layout.halo_cells.size
        f64 = dict(dtype=torch.float64, device=dev)
        self.zext = torch.zeros(nfo + nco + nhf + nhc, **f64)      # [own | halo f | halo c]
        self.tf_ext = torch.zeros(nfo + nhf, **f64)
        self.yc_ext = torch.zeros(nco + nhc, **f64)
        self.uc = torch.zeros(max(nco, 1), **f64)
        self.af = torch.zeros(max(nfo, 1), **f64)
        self.ic = self.ilu = None
        self.s1 = None

    # -- setup ------------------------------------------------------------
    def build(self) -> None:
        """Stage 1 on the extended subsystem, block-Jacobi stage 2 + factors."""
        from .device import DeviceCsr
        from .patterns import static_patterns_device
        from .precond import build_stage1
        o = self.opts
        lib, c = self.lib, self.ctx
        if o["dynamic"] is not None:
            s1 = build_stage1(self.ext, dynamic=o["dynamic"], tau_filt=o["tau_filt"],
                              filtration=o["filtration"], face_drop_tol=o["face_drop_tol"], no_fill=o["no_fill"])
        else:
            pats = (static_patterns_device(self.ext.topology, o["prototype"]) if o["kind"] == "static"
                    else None)
            if pats is None:
                from .patterns import base_pattern
                pats = base_pattern(self.ext.A_cf)
            s1 = build_stage1(self.ext, patterns=pats, tau_filt=o["tau_filt"], filtration=o["filtration"],
                              face_drop_tol=o["face_drop_tol"], no_fill=o["no_fill"])
        self.s1 = s1
        H = s1._part(L.S1_H)
        lay = self.layout
        h = C.c_void_p()
        L.check(lib.edfa_csr_submatrix(c, H.handle, lay.n_cells, C.c_void_p(self.own_in_ext.data_ptr()),
                                       C.c_void_p(self.cell_map.data_ptr()), lay.n_cells, C.byref(h)))
        H_own = DeviceCsr(h)
        tau = o["tau_filt"] if o["filtration"] == "post-schur" else 0.0
        h = C.c_void_p()
        L.check(lib.edfa_csr_sub(c, self.A_cc_own.handle, H_own.handle, tau, C.byref(h)))
        self.S_own = DeviceCsr(h)
        nx, ny, _ = lay.nxyz
        self._free_factors()
        nf = int(bool(o["no_fill"]))
        f = C.c_void_p()
        L.check(lib.edfa_factor_ilu(c, self.S_own.handle, o["schur_drop_tol"], nf, nx, ny, lay.k1 - lay.k0,
                                    C.byref(f)))
        self.ilu = f
        f = C.c_void_p()
        L.check(lib.edfa_factor_ic(c, self.A_ff_own.handle, o["face_drop_tol"], nf, C.byref(f)))
        self.ic = f

    def _free_factors(self):
        for name in ("ic", "ilu"):
            f = getattr(self, name, None)
            if f:
                L.check(self.lib.edfa_factor_destroy(f))
                setattr(self, name, None)

    def __del__(self):
        try:
            if L._lib is not None:
                self._free_factors()
        except Exception:   # pragma: no cover
            pass

    # -- vector kernels ----------------------------------------------------
    def empty(self, *shape):
        return torch.empty(*shape, dtype=torch.float64, device=self.rhs.device)

    def gather(self, src, kind, q):
        idx = self.send[(kind, q)]
        out = self.empty(idx.numel())
        L.check(self.lib.edfa_gather(self.ctx, idx.numel(), C.c_void_p(idx.data_ptr()),
                                     C.c_void_p(src.data_ptr()), C.c_void_p(out.data_ptr())))
        return out

    def multidot(self, V, nvec, w, out):
        n = self.layout.n_own
        L.check(self.lib.edfa_multidot(self.ctx, n, nvec, C.c_void_p(V.data_ptr()), V.stride(0),
                                       C.c_void_p(w.data_ptr()), C.c_void_p(out.data_ptr())))

    def multiaxpy(self, V, nvec, h, w_in, out, norm2):
        n = self.layout.n_own
        L.check(self.lib.edfa_multiaxpy(self.ctx, n, nvec, C.c_void_p(V.data_ptr()), V.stride(0),
                                        C.c_void_p(h.data_ptr()), 1.0,
                                        None if w_in is None else C.c_void_p(w_in.data_ptr()),
                                        C.c_void_p(out.data_ptr()),
                                        None if norm2 is None else C.c_void_p(norm2.data_ptr())))

    def sync(self):
        L.check(self.lib.edfa_ctx_sync(self.ctx))

    def axpby(self, a, x, b, y):
        L.check(self.lib.edfa_axpby(self.ctx, y.numel(), a, C.c_void_p(x.data_ptr()), b,
                                    C.c_void_p(y.data_ptr())))

    # DCGS2 building blocks (krylov.cu): local dots, coefficients from the summed
    # dots, local two-output update
    def dcgs2_dots(self, V, j, out):
        L.check(self.lib.edfa_dcgs2_dots(self.ctx, self.layout.n_own, j, C.c_void_p(V.data_ptr()), V.stride(0),
                                         C.c_void_p(out.data_ptr())))

    def dcgs2_coeffs(self, j, m, dots, H, h1, coef, hcol):
        L.check(self.lib.edfa_dcgs2_coeffs(self.ctx, j, m, C.c_void_p(dots.data_ptr()), C.c_void_p(H.data_ptr()),
                                           C.c_void_p(h1.data_ptr()), C.c_void_p(coef.data_ptr()),
                                           C.c_void_p(hcol.data_ptr())))

    def dcgs2_update(self, V, j, coef):
        L.check(self.lib.edfa_dcgs2_update(self.ctx, self.layout.n_own, j, C.c_void_p(V.data_ptr()), V.stride(0),
                                           C.c_void_p(coef.data_ptr())))

    def fetch(self, t):
        """Asynchronous device->host copy of t; returns a callable giving the array."""
        host = torch.empty(t.shape, dtype=t.dtype, pin_memory=True)
        host.copy_(t, non_blocking=True)
        ev = torch.cuda.Event()
        ev.record()
        return lambda: (ev.synchronize(), host.numpy())[1]

    def copy(self, src, dst):
        self.axpby(1.0, src, 0.0, dst)

    # -- operator pieces ---------------------------------------------------
    def spmv_ext(self, y):
        """y = A_loc zext (zext's own part and halo already in place)."""
        L.check(self.lib.edfa_spmv(self.ctx, self.A_loc.handle, C.c_void_p(self.zext.data_ptr()),
                                   C.c_void_p(y.data_ptr()), 1.0, 0.0))

    def spmv_interior(self, y):
        """y = A_loc zext on the rows without halo columns (0 on the others)."""
        L.check(self.lib.edfa_spmv(self.ctx, self.A_int.handle, C.c_void_p(self.zext.data_ptr()),
                                   C.c_void_p(y.data_ptr()), 1.0, 0.0))

    def spmv_boundary(self, y):
        """The rows that read halo values, after the exchange."""
        if self.brows.numel():
            L.check(self.lib.edfa_spmv_rows(self.ctx, self.A_bnd.handle, C.c_void_p(self.brows.data_ptr()),
                                            C.c_void_p(self.zext.data_ptr()), C.c_void_p(y.data_ptr())))

    def apply_faces(self, r):
        """t_f = -(L L^T)^-1 r_f into tf_ext[:nfo]."""
        nfo = self.layout.n_faces
        if nfo:
            L.check(self.lib.edfa_factor_solve(self.ctx, self.ic, C.c_void_p(r.data_ptr()), -1.0,
                                               C.c_void_p(self.tf_ext.data_ptr())))

    def apply_cells(self, r):
        """y_c = (L U)^-1 (r_c - A_cf t_f) into yc_ext[:nco]."""
        nfo, nco = self.layout.n_faces, self.layout.n_cells
        if not nco:
            return
        rc = r[nfo:]
        self.copy(rc, self.uc[:nco])
        L.check(self.lib.edfa_spmv(self.ctx, self.A_cf_loc.handle, C.c_void_p(self.tf_ext.data_ptr()),
                                   C.c_void_p(self.uc.data_ptr()), -1.0, 1.0))
        L.check(self.lib.edfa_factor_solve(self.ctx, self.ilu, C.c_void_p(self.uc.data_ptr()), 1.0,
                                           C.c_void_p(self.yc_ext.data_ptr())))

    def apply_finish(self, y):
        """y = [t_f + (L L^T)^-1 A_fc y_c ; y_c]."""
        nfo, nco = self.layout.n_faces, self.layout.n_cells
        if nfo:
            L.check(self.lib.edfa_spmv(self.ctx, self.A_fc_loc.handle, C.c_void_p(self.yc_ext.data_ptr()),
                                       C.c_void_p(self.af.data_ptr()), 1.0, 0.0))
            L.check(self.lib.edfa_factor_solve(self.ctx, self.ic, C.c_void_p(self.af.data_ptr()), 1.0,
                                               C.c_void_p(y.data_ptr())))
            self.axpby(1.0, self.tf_ext[:nfo], 1.0, y[:nfo])
        if nco:
            self.copy(self.yc_ext[:nco], y[nfo:nfo + nco])


# ---------------------------------------------------------------------------
# distributed operator + GMRES

class CommTimer:
    """CUDA events around the communication calls of a distributed solve
    (halo exchanges, all-reduces) on the current stream: device time spent
    inside NCCL, reported as a share of the step (bench.py)."""

    def __init__(self):
        self.pairs = {"halo": [], "allreduce": []}
        self.enabled = False

    def __call__(self, kind):
        timer = self

        class _Span:
            def __enter__(self_):
                if timer.enabled:
                    self_.e0 = torch.cuda.Event(enable_timing=True)
                    self_.e0.record()

            def __exit__(self_, *exc):
                if timer.enabled:
                    e1 = torch.cuda.Event(enable_timing=True)
                    e1.record()
                    timer.pairs[kind].append((self_.e0, e1))
        return _Span()

    def collect(self, reset=True):
        torch.cuda.synchronize()
        out = {k: sum(a.elapsed_time(b) for a, b in v) for k, v in self.pairs.items()}
        out.update({f"{k}_calls": len(v) for k, v in self.pairs.items()})
        if reset:
            self.pairs = {k: [] for k in self.pairs}
        return out


class SlabOperator:
    """The block operator and the EDFA preconditioner over a set of slabs."""

    def __init__(self, parts, comm):
        self.parts = parts
        self.comm = comm
        self.halo = HaloExchange(parts, comm)
        self.timer = CommTimer()

    def _own_views(self, vecs, kind):
        out = []
        for p, v in zip(self.parts, vecs):
            nfo = p.layout.n_faces
            out.append(v[:nfo] if kind == "f" else v[nfo:p.layout.n_own])
        return out

    def precond_into_zext(self, rs):
        """zext[:n_own] = P^-1 r per part (two halo exchanges)."""
        for p, r in zip(self.parts, rs):
            p.apply_faces(r)
        with self.timer("halo"):
            self.halo.run("f", [p.tf_ext[:p.layout.n_faces] for p in self.parts],
                          [p.tf_ext[p.layout.n_faces:] for p in self.parts])
        for p, r in zip(self.parts, rs):
            p.apply_cells(r)
        with self.timer("halo"):
            self.halo.run("c", [p.yc_ext[:p.layout.n_cells] for p in self.parts],
                          [p.yc_ext[p.layout.n_cells:] for p in self.parts])
        for p in self.parts:
            p.apply_finish(p.zext[:p.layout.n_own])

    def matvec_zext(self, ws):
        """w = A zext per part (exchanges the halo of zext's own part)."""
        with self.timer("halo"):
            works = self.halo.start_many([
                ("f", [p.zext[:p.layout.n_faces] for p in self.parts],
                 [p.zext[p.layout.n_own:p.layout.n_own + p.layout.halo_faces.size] for p in self.parts]),
                ("c", [p.zext[p.layout.n_faces:p.layout.n_own] for p in self.parts],
                 [p.zext[p.layout.n_own + p.layout.halo_faces.size:] for p in self.parts])])
        for p, w in zip(self.parts, ws):          # interior rows overlap the exchange
            p.spmv_interior(w)
        with self.timer("halo"):
            self.comm.p2p_wait(works)
        for p, w in zip(self.parts, ws):          # rows that read halo values
            p.spmv_boundary(w)

    def allsum(self, partials):
        t = partials[0]
        if len(partials) > 1:
            t = partials[0].clone()
            for q in partials[1:]:
                t += q.to(t.device)
        with self.timer("allreduce"):
            self.comm.allreduce_(t)
        return t


def slab_gmres(op: SlabOperator, bs, tol=1e-8, restart=50, max_it=2000):
    """Right-preconditioned restarted GMRES(m) on slab-distributed vectors.

    The same algorithm as the single-device solver (krylov.cu gmres): x0 = 0,
    DCGS2 Arnoldi -- per step one local dot kernel, ONE all-reduce of the
    2(j+1) dot products over the slabs (NCCL over NVLink between GPUs), the
    coefficient kernel on the summed dots and one local two-output update --
    and the host one step behind the devices (it reads Hessenberg column j-1
    while step j+1 is queued), Givens rotations on the host, convergence
    confirmed on the true residual (hx/krylov.py conventions).
    Returns (list of local x, SolveReport)."""
    if tol <= 0:
        raise ValueError("tol must be positive")
    if not 1 <= restart <= 62:
        raise ValueError("restart must be in [1, 62]")
    parts = op.parts
    m = restart
    rep = SolveReport()
    hd = [p.empty(192).zero_() for p in parts]

    def global_dot(xs, ys):
        for p, x, y, h in zip(parts, xs, ys, hd):
            p.multidot(x.view(1, -1), 1, y, h[128:129])
        return float(op.allsum([h[128:129] for h in hd]).item())

    bnorm = math.sqrt(global_dot(bs, bs))
    xs = [p.empty(p.layout.n_own).zero_() for p in parts]
    if bnorm == 0.0:
        rep.converged, rep.final_relres = True, 0.0
        rep.relres_history.append(0.0)
        return xs, rep
    V = [p.empty(m + 2, p.layout.n_own) for p in parts]
    Hd = [p.empty(m, m + 1).zero_() for p in parts]        # unrotated Hessenberg, column i = row i
    h1 = [p.empty(64).zero_() for p in parts]
    coef = [p.empty(192).zero_() for p in parts]
    dots = [p.empty(128).zero_() for p in parts]
    hcol = [p.empty(2, 64).zero_() for p in parts]
    rs = [b.clone() for b in bs]
    beta = bnorm
    happy = False
    pending = {}

    def enqueue_step(st):
        op.precond_into_zext([v[st] for v in V])
        op.matvec_zext([v[st + 1] for v in V])
        for p, v, d in zip(parts, V, dots):
            p.dcgs2_dots(v, st, d)
        dsum = op.allsum(dots)
        for i, p in enumerate(parts):
            p.dcgs2_coeffs(st, m, dsum.to(dots[i].device), Hd[i], h1[i], coef[i], hcol[i][st & 1])
        for p, v, cf in zip(parts, V, coef):
            p.dcgs2_update(v, st, cf)
        if st >= 1:
            pending[st] = parts[0].fetch(hcol[0][st & 1][:st + 1])

    while rep.n_it < max_it:
        for p, v, r in zip(parts, V, rs):
            p.axpby(1.0 / beta, r, 0.0, v[0])
        H = np.zeros((m + 1, m))
        cs, sn, g = np.zeros(m), np.zeros(m), np.zeros(m + 1)
        g[0] = beta
        k = 0
        budget = min(m, max_it - rep.n_it)     # columns this cycle (step s finalises column s-1)
        enq = 0
        pending.clear()
        enqueue_step(enq)
        enq += 1
        enqueue_step(enq)
        enq += 1
        for j in range(budget):
            if enq <= budget:
                enqueue_step(enq)              # keep one step ahead of the host
                enq += 1
            col = pending.pop(j + 1)()
            rep.n_it += 1
            H[:j + 2, j] = col[:j + 2]
            wn = col[j + 1]
            for i in range(j):
                a, c = H[i, j], H[i + 1, j]
                H[i, j] = cs[i] * a + sn[i] * c
                H[i + 1, j] = -sn[i] * a + cs[i] * c
            den = math.hypot(H[j, j], H[j + 1, j])
            cs[j], sn[j] = (1.0, 0.0) if den == 0.0 else (H[j, j] / den, H[j + 1, j] / den)
            H[j, j], H[j + 1, j] = den, 0.0
            g[j + 1] = -sn[j] * g[j]
            g[j] = cs[j] * g[j]
            est = abs(g[j + 1]) / bnorm
            rep.relres_history.append(est)
            k = j + 1
            if wn == 0.0:
                happy = True
                break
            if est <= tol:
                break
        # queued speculative steps only write rows >= k + 1
        y = np.zeros(k)
        for i in range(k - 1, -1, -1):
            s = g[i] - H[i, i + 1:k] @ y[i + 1:k]
            y[i] = s / H[i, i] if H[i, i] != 0.0 else 0.0
        yd = [torch.from_numpy(y.copy()).to(h.device) for h in hd]
        for p, v, r, yy in zip(parts, V, rs, yd):
            p.multiaxpy(v, k, yy, None, r, None)                  # r <- V y (scratch)
        op.precond_into_zext(rs)
        for p, x in zip(parts, xs):
            p.axpby(1.0, p.zext[:p.layout.n_own], 1.0, x)
        for p, x in zip(parts, xs):
            p.copy(x, p.zext[:p.layout.n_own])
        op.matvec_zext(rs)
        for p, r, b in zip(parts, rs, bs):
            p.axpby(1.0, b, -1.0, r)                              # r = b - A x
        beta = math.sqrt(global_dot(rs, rs))
        for p in parts:        # once per restart cycle: a triangular solve that hit its spin limit raises
            p.sync()
        if beta / bnorm <= tol:
            rep.converged = True
            break
        if happy or beta == 0.0:
            rep.breakdown = True
            break
    rep.final_relres = beta / bnorm
    if rep.n_it == 0:
        rep.relres_history.append(beta / bnorm)
    return xs, rep


class SlabSolver:
    """Build + solve over the slabs this process holds (drop-in counterpart
    of ``BlockLDUPreconditioner.build`` + ``gmres`` for a partitioned run)."""

    def __init__(self, layouts, comm, **opts):
        self.layouts = layouts
        self.comm = comm
        self.parts = [CudaSlab(lay, **opts) for lay in layouts]
        self.op = SlabOperator(self.parts, comm)

    def build(self):
        for p in self.parts:
            p.build()

    def solve(self, tol=1e-8, restart=50, max_it=2000):
        return slab_gmres(self.op, [p.rhs for p in self.parts], tol=tol, restart=restart, max_it=max_it)
