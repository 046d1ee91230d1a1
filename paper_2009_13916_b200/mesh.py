"""Hexahedral box grids, per-cell conductivity tensors, rock properties and
boundary specifications -- the input producer that feeds the EDFA path.

This is harness-side code: it generates the seeded
synthetic grids of BASELINE.json's five configurations on the GPU box, where
the reference package is not available.  Numbering conventions follow the
reference exactly so the assembled blocks are interchangeable with hexflow's:

* cells x-fastest, ``e = i + nx*(j + ny*k)``            (hx/grid.py:49-50)
* faces grouped by family (x, y, z), each k-slowest      (hx/grid.py:97-107)
* local face slots (-x, +x, -y, +y, -z, +z)              (hx/grid.py:109-113)
* a face is owned by its lower-indexed cell              (hx/grid.py:121-129)

Everything is vectorised numpy; no per-cell Python loops.
"""

from __future__ import annotations

import dataclasses
from dataclasses import dataclass

import numpy as np

AXIS_TAGS = ("x-", "x+", "y-", "y+", "z-", "z+")

# reference-cube corner signs, node order of hx/refelem.py:13-16
_CORNERS = np.array([[-1, -1, -1], [1, -1, -1], [1, 1, -1], [-1, 1, -1],
                     [-1, -1, 1], [1, -1, 1], [1, 1, 1], [-1, 1, 1]], float)
# corner nodes of each local face (hx/refelem.py:19-26)
FACE_CORNERS = np.array([[0, 3, 7, 4], [1, 2, 6, 5], [0, 1, 5, 4],
                         [3, 2, 6, 7], [0, 1, 2, 3], [4, 5, 6, 7]])
_G = 1.0 / np.sqrt(3.0)


def gauss3():
    """2x2x2 Gauss points (x fastest) with unit weights."""
    pts = np.array([[a * _G, b * _G, c * _G]
                    for c in (-1, 1) for b in (-1, 1) for a in (-1, 1)])
    return pts, np.ones(8)


def shape_grad(xi):
    """dN_a/dxi_b of the trilinear map at one point, shape (8, 3)."""
    s = _CORNERS
    f = 1.0 + xi[None, :] * s
    g = np.empty((8, 3))
    g[:, 0] = s[:, 0] * f[:, 1] * f[:, 2] / 8.0
    g[:, 1] = s[:, 1] * f[:, 0] * f[:, 2] / 8.0
    g[:, 2] = s[:, 2] * f[:, 0] * f[:, 1] / 8.0
    return g


def rt0_reference(xi):
    """Reference RT0 basis (6 faces x 3 components) at one point."""
    out = np.zeros((6, 3))
    for ax in range(3):
        out[2 * ax, ax] = (xi[ax] - 1.0) / 8.0
        out[2 * ax + 1, ax] = (xi[ax] + 1.0) / 8.0
    return out


@dataclass(frozen=True)
class HexGrid:
    """Topology + geometry of an nx*ny*nz hexahedral box (hx/grid.py:22-65)."""

    nx: int
    ny: int
    nz: int
    node_coords: np.ndarray
    elem_to_nodes: np.ndarray
    elem_to_faces: np.ndarray
    face_to_elems: np.ndarray
    face_local: np.ndarray
    face_area: np.ndarray
    elem_volume: np.ndarray

    @property
    def n_elems(self) -> int:
        return self.elem_to_faces.shape[0]

    @property
    def n_faces(self) -> int:
        return self.face_to_elems.shape[0]

    @property
    def boundary_faces(self) -> np.ndarray:
        return np.flatnonzero(self.face_to_elems[:, 1] < 0)

    def elem_index(self, i, j, k) -> int:
        return int(i + self.nx * (j + self.ny * k))

    def neighbor(self, e: int, slot: int) -> int:
        a, b = self.face_to_elems[self.elem_to_faces[e, slot]]
        return int(b if a == e else a)

    def neighbors(self) -> np.ndarray:
        """(n_elems, 6) cell across each local face, -1 on the hull."""
        fe = self.face_to_elems[self.elem_to_faces]          # (n, 6, 2)
        me = np.arange(self.n_elems)[:, None]
        return np.where(fe[:, :, 0] == me, fe[:, :, 1], fe[:, :, 0])

    def elem_coords(self) -> np.ndarray:
        return self.node_coords[self.elem_to_nodes]


def _topology(nx, ny, nz):
    cells = np.arange(nx * ny * nz)
    ci = cells % nx
    cj = (cells // nx) % ny
    ck = cells // (nx * ny)

    def node(i, j, k):
        return i + (nx + 1) * (j + (ny + 1) * k)

    e2n = np.stack([node(ci, cj, ck), node(ci + 1, cj, ck),
                    node(ci + 1, cj + 1, ck), node(ci, cj + 1, ck),
                    node(ci, cj, ck + 1), node(ci + 1, cj, ck + 1),
                    node(ci + 1, cj + 1, ck + 1), node(ci, cj + 1, ck + 1)],
                   axis=1).astype(np.int64)
    nxf = (nx + 1) * ny * nz
    nyf = nx * (ny + 1) * nz
    fx = lambda i, j, k: i + (nx + 1) * (j + ny * k)                # noqa: E731
    fy = lambda i, j, k: nxf + i + nx * (j + (ny + 1) * k)           # noqa: E731
    fz = lambda i, j, k: nxf + nyf + i + nx * (j + ny * k)           # noqa: E731
    e2f = np.stack([fx(ci, cj, ck), fx(ci + 1, cj, ck),
                    fy(ci, cj, ck), fy(ci, cj + 1, ck),
                    fz(ci, cj, ck), fz(ci, cj, ck + 1)], axis=1).astype(np.int64)
    n_faces = nxf + nyf + nx * ny * (nz + 1)
    f2e = np.full((n_faces, 2), -1, dtype=np.int64)
    floc = np.full((n_faces, 2), -1, dtype=np.int64)
    # the lower-indexed cell sees an interior face at a "+" slot: it owns it
    for slot in (1, 3, 5):
        f2e[e2f[:, slot], 0] = cells
        floc[e2f[:, slot], 0] = slot
    for slot in (0, 2, 4):
        f = e2f[:, slot]
        unowned = f2e[f, 0] < 0
        f2e[f[unowned], 0] = cells[unowned]
        floc[f[unowned], 0] = slot
        f2e[f[~unowned], 1] = cells[~unowned]
        floc[f[~unowned], 1] = slot
    return e2n, e2f, f2e, floc


_CHUNK = 1 << 20   # cells / faces per block of the geometry pass (bounded temporaries at 256^3)


def geometry(node_coords, e2n, f2e, floc):
    """Cell volumes (2x2x2 Gauss) and owner-side bilinear face areas
    (hx/grid.py:137-164).  Raises ValueError on an inverted cell.

    Same quadrature and accumulation order as the reference; per block of
    cells, the Jacobian entries of all eight points come from three GEMMs with
    contiguous (point, entry) rows, so a 256^3 grid takes seconds instead of
    minutes (values agree to the last bits, inside the 1e-13 assembly
    tolerance)."""
    pts, wts = gauss3()
    dNT = np.concatenate([shape_grad(p) for p in pts], axis=1).T.copy()   # (8 points * 3, 8 nodes)
    n_e = e2n.shape[0]
    vol = np.zeros(n_e)
    for c0 in range(0, n_e, _CHUNK):
        c1 = min(c0 + _CHUNK, n_e)
        nodes = e2n[c0:c1].T                                                 # (8, c)
        J = [dNT @ node_coords[nodes, a] for a in range(3)]                 # J[a][3q + b] = dx_a/dxi_b at q
        acc = np.zeros(c1 - c0)
        for q, w in enumerate(wts):
            (a0, a1, a2), (b0, b1, b2), (d0, d1, d2) = (J[a][3 * q:3 * q + 3] for a in range(3))
            det = a0 * (b1 * d2 - b2 * d1) - a1 * (b0 * d2 - b2 * d0) + a2 * (b0 * d1 - b1 * d0)
            if np.any(det <= 0):
                raise ValueError(f"cell {c0 + int(np.flatnonzero(det <= 0)[0])} is inverted")
            acc += w * det
        vol[c0:c1] = acc
    n_f = f2e.shape[0]
    area = np.zeros(n_f)
    dUV = []
    for v in (-_G, _G):
        for u in (-_G, _G):
            dUV.append(np.array([-(1 - v), (1 - v), (1 + v), -(1 + v)]) / 4.0)
            dUV.append(np.array([-(1 - u), -(1 + u), (1 + u), (1 - u)]) / 4.0)
    dUVT = np.stack(dUV, axis=0)                                             # (8, 4 corners)
    for c0 in range(0, n_f, _CHUNK):
        c1 = min(c0 + _CHUNK, n_f)
        fn = e2n[f2e[c0:c1, 0][:, None], FACE_CORNERS[floc[c0:c1, 0]]].T     # (4, c)
        R = [dUVT @ node_coords[fn, a] for a in range(3)]                   # R[a][2q + (u|v)]
        acc = np.zeros(c1 - c0)
        for q in range(4):
            (ux, vx), (uy, vy), (uz, vz) = (R[a][2 * q:2 * q + 2] for a in range(3))
            cx = uy * vz - uz * vy
            cy = uz * vx - ux * vz
            cz = ux * vy - uy * vx
            acc += np.sqrt(cx * cx + cy * cy + cz * cz)
        area[c0:c1] = acc
    return vol, area


def box_grid(nx, ny, nz, dx, dy, dz, z0_layer: int = 0) -> HexGrid:
    """Regular nx*ny*nz box with spacings dx, dy, dz (hx/grid.py:68-134).

    ``z0_layer`` > 0 builds the cell layers [z0, z0 + nz) of a taller box
    (a z-slab of the multi-GPU partition): node z = (k + z0) dz exactly as
    in the full box, so the slab's geometry is the full box's bit for bit."""
    if min(nx, ny, nz) < 1 or min(dx, dy, dz) <= 0:
        raise ValueError("grid dimensions must be >= 1 and spacings > 0")
    nx, ny, nz = int(nx), int(ny), int(nz)
    n = np.arange((nx + 1) * (ny + 1) * (nz + 1))
    coords = np.stack([(n % (nx + 1)) * dx,
                       ((n // (nx + 1)) % (ny + 1)) * dy,
                       (n // ((nx + 1) * (ny + 1)) + int(z0_layer)) * dz], axis=1).astype(float)
    e2n, e2f, f2e, floc = _topology(nx, ny, nz)
    vol, area = geometry(coords, e2n, f2e, floc)
    return HexGrid(nx, ny, nz, coords, e2n, e2f, f2e, floc, area, vol)


def with_nodes(grid: HexGrid, coords: np.ndarray) -> HexGrid:
    """Same topology, new node coordinates, geometry recomputed."""
    vol, area = geometry(coords, grid.elem_to_nodes, grid.face_to_elems,
                         grid.face_local)
    return dataclasses.replace(grid, node_coords=coords, elem_volume=vol,
                               face_area=area)


def perturb_interior(grid: HexGrid, frac: float, seed: int) -> HexGrid:
    """Config 3 distortion: every node not on a boundary plane moves by
    U(-frac*h, frac*h) per coordinate (h = the local spacing)."""
    nx, ny, nz = grid.nx, grid.ny, grid.nz
    c = grid.node_coords.copy()
    n = np.arange(c.shape[0])
    i = n % (nx + 1)
    j = (n // (nx + 1)) % (ny + 1)
    k = n // ((nx + 1) * (ny + 1))
    inner = (i > 0) & (i < nx) & (j > 0) & (j < ny) & (k > 0) & (k < nz)
    h = np.array([c[1, 0] - c[0, 0],
                  c[nx + 1, 1] - c[0, 1],
                  c[(nx + 1) * (ny + 1), 2] - c[0, 2]])
    rng = np.random.default_rng(seed)
    d = rng.uniform(-frac, frac, size=(int(inner.sum()), 3)) * h[None, :]
    c[inner] += d
    return with_nodes(grid, c)


# ---------------------------------------------------------------------------
# fields and properties

@dataclass(frozen=True)
class Conductivity:
    """Per-cell SPD conductivity tensors (n, 3, 3) -- hx/grid.py:209-239."""

    tensors: np.ndarray

    @classmethod
    def homogeneous(cls, n, kx, ky=None, kz=None):
        t = np.zeros((n, 3, 3))
        t[:, 0, 0] = kx
        t[:, 1, 1] = kx if ky is None else ky
        t[:, 2, 2] = kx if kz is None else kz
        return cls(t)

    @classmethod
    def diagonal(cls, kx, ky, kz):
        kx = np.asarray(kx, float)
        t = np.zeros((kx.size, 3, 3))
        t[:, 0, 0], t[:, 1, 1], t[:, 2, 2] = kx, ky, kz
        return cls(t)


def loguniform_field(grid: HexGrid, seed: int, lo: float, hi: float) -> Conductivity:
    """hx/grid.py:242-256 "loguniform" mode (isotropic, one draw per cell)."""
    rng = np.random.default_rng(seed)
    k = 10.0 ** rng.uniform(np.log10(lo), np.log10(hi), size=grid.n_elems)
    return Conductivity.diagonal(k, k, k)


@dataclass(frozen=True)
class RockProps:
    """gamma [bar/m], compressibilities [1/bar], porosity (hx/grid.py:352-376)."""

    gamma: float = 0.101
    alpha: float = 4.67e-5
    beta: float = 4.84e-5
    porosity: float = 0.2

    def storage(self, n) -> np.ndarray:
        phi = np.full(n, float(self.porosity))
        return self.gamma * (self.alpha + phi * self.beta)


@dataclass
class Boundaries:
    """Dirichlet planes / Neumann planes / full-thickness well columns
    (hx/grid.py:396-430)."""

    pressure_planes: dict = dataclasses.field(default_factory=dict)
    flux_planes: dict = dataclasses.field(default_factory=dict)
    wells: list = dataclasses.field(default_factory=list)   # (i, j, p)

    def resolve(self, grid: HexGrid):
        """Returns (dir_faces, dir_vals, neu_faces, neu_vals), faces sorted."""
        bnd = grid.boundary_faces
        slot_of = grid.face_local[bnd, 0]
        dmap: dict[int, float] = {}
        for tag, p in self.pressure_planes.items():
            for f in bnd[slot_of == AXIS_TAGS.index(tag)]:
                dmap[int(f)] = float(p)
        for (i, j, p) in self.wells:
            if not (0 <= i < grid.nx and 0 <= j < grid.ny):
                raise ValueError(f"well column ({i}, {j}) outside grid")
            cells = i + grid.nx * (j + grid.ny * np.arange(grid.nz))
            for f in np.unique(grid.elem_to_faces[cells][:, :4]):
                dmap[int(f)] = float(p)
        nmap: dict[int, float] = {}
        for tag, v in self.flux_planes.items():
            for f in bnd[slot_of == AXIS_TAGS.index(tag)]:
                nmap[int(f)] = float(v)
        if set(dmap) & set(nmap):
            raise ValueError("a face has both a prescribed pressure and a flux")
        df = np.array(sorted(dmap), dtype=np.int64)
        nf = np.array(sorted(nmap), dtype=np.int64)
        return (df, np.array([dmap[f] for f in df.tolist()], float),
                nf, np.array([nmap[f] for f in nf.tolist()], float))
