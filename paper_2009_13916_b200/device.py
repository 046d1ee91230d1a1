"""Device-resident matrices and block systems behind the drop-in API.

PyTorch supplies the CUDA stream and the memory of vectors; matrices live in
libedfa-owned device memory (stream-ordered pool) and are addressed through
opaque handles.  Nothing here computes: every operation is a libedfa call.
"""

from __future__ import annotations

import ctypes as C

import numpy as np
import scipy.sparse as sp
import torch

from . import _lib as L

_CTX: dict[int, C.c_void_p] = {}


def ctx(device: int | None = None) -> C.c_void_p:
    """Context for a CUDA device, bound to torch's current stream."""
    if not torch.cuda.is_available():
        raise RuntimeError("the EDFA path needs a CUDA device (there is no CPU fallback)")
    dev = torch.cuda.current_device() if device is None else int(device)
    lib = L.lib()
    h = _CTX.get(dev)
    stream = torch.cuda.current_stream(dev).cuda_stream
    if h is None:
        h = C.c_void_p()
        with torch.cuda.device(dev):
            L.check(lib.edfa_ctx_create(dev, C.c_void_p(stream), C.byref(h)))
        _CTX[dev] = h
    else:
        L.check(lib.edfa_ctx_set_stream(h, C.c_void_p(stream)))
    return h


class option:
    """Context manager selecting one of libedfa's algorithm alternatives on the
    current device's context (edfa_ctx_set_option; names in include/edfa.h),
    restoring the previous value on exit -- the A/B switch the tests use."""

    def __init__(self, name: str, value: int):
        self.name, self.value = name.encode(), int(value)

    def __enter__(self):
        c = ctx()
        old = C.c_int32()
        L.check(L.lib().edfa_ctx_get_option(c, self.name, C.byref(old)))
        self.old = old.value
        L.check(L.lib().edfa_ctx_set_option(c, self.name, self.value))
        return self

    def __exit__(self, *exc):
        L.check(L.lib().edfa_ctx_set_option(ctx(), self.name, self.old))


def dptr(t: torch.Tensor) -> C.c_void_p:
    return C.c_void_p(t.data_ptr())


def as_device_vector(v, n=None) -> torch.Tensor:
    """float64 contiguous CUDA tensor (copies host arrays)."""
    if isinstance(v, torch.Tensor):
        t = v.to(device="cuda", dtype=torch.float64)
    else:
        t = torch.from_numpy(np.ascontiguousarray(np.asarray(v, dtype=np.float64))).to("cuda")
    t = t.contiguous()
    if n is not None and t.numel() != n:
        raise ValueError(f"shape mismatch: expected {n} entries, got {t.numel()}")
    return t


class DeviceCsr:
    """A CSR matrix in libedfa device memory (int32 indices, float64 values)."""

    def __init__(self, handle: C.c_void_p, owner: bool = True, keepalive=None):
        self.handle = handle
        self._owner = owner
        self._keep = keepalive
        r, c, z = C.c_int32(), C.c_int32(), C.c_int64()
        L.check(L.lib().edfa_csr_info(handle, C.byref(r), C.byref(c), C.byref(z)))
        self.shape = (r.value, c.value)
        self.nnz = z.value

    @classmethod
    def from_scipy(cls, A) -> "DeviceCsr":
        A = sp.csr_matrix(A)
        if A.nnz >= 2 ** 31:
            raise ValueError("matrix exceeds 2^31-1 stored entries")
        ptr = np.ascontiguousarray(A.indptr, dtype=np.int32)
        idx = np.ascontiguousarray(A.indices, dtype=np.int32)
        val = np.ascontiguousarray(A.data, dtype=np.float64)
        h = C.c_void_p()
        L.check(L.lib().edfa_csr_create(ctx(), A.shape[0], A.shape[1], A.nnz,
                                         ptr.ctypes.data_as(C.c_void_p), idx.ctypes.data_as(C.c_void_p),
                                         val.ctypes.data_as(C.c_void_p), L.MEM_HOST, C.byref(h)))
        return cls(h)

    @classmethod
    def from_arrays(cls, shape, indptr, indices, data=None, device: bool = False) -> "DeviceCsr":
        """Pattern-only when data is None.  Arrays are host numpy or CUDA tensors."""
        h = C.c_void_p()
        if device:
            ptr = indptr.to(torch.int32).contiguous()
            idx = indices.to(torch.int32).contiguous()
            val = None if data is None else data.to(torch.float64).contiguous()
            L.check(L.lib().edfa_csr_create(ctx(), shape[0], shape[1], idx.numel(), dptr(ptr), dptr(idx),
                                             None if val is None else dptr(val), L.MEM_DEVICE, C.byref(h)))
            torch.cuda.current_stream().synchronize()
        else:
            ptr = np.ascontiguousarray(indptr, dtype=np.int32)
            idx = np.ascontiguousarray(indices, dtype=np.int32)
            val = None if data is None else np.ascontiguousarray(data, dtype=np.float64)
            L.check(L.lib().edfa_csr_create(ctx(), shape[0], shape[1], idx.size,
                                             ptr.ctypes.data_as(C.c_void_p), idx.ctypes.data_as(C.c_void_p),
                                             None if val is None else val.ctypes.data_as(C.c_void_p),
                                             L.MEM_HOST, C.byref(h)))
        return cls(h)

    def arrays(self, values: bool = True):
        n = self.shape[0]
        ptr = np.empty(n + 1, dtype=np.int32)
        idx = np.empty(self.nnz, dtype=np.int32)
        val = np.empty(self.nnz, dtype=np.float64) if values else None
        L.check(L.lib().edfa_csr_export(ctx(), self.handle, ptr.ctypes.data_as(C.c_void_p),
                                         idx.ctypes.data_as(C.c_void_p),
                                         None if val is None else val.ctypes.data_as(C.c_void_p), L.MEM_HOST))
        return ptr, idx, val

    def to_scipy(self) -> sp.csr_matrix:
        ptr, idx, val = self.arrays(True)
        return sp.csr_matrix((val, idx, ptr), shape=self.shape)

    def matvec(self, x: torch.Tensor, y: torch.Tensor | None = None, alpha=1.0, beta=0.0) -> torch.Tensor:
        x = as_device_vector(x, self.shape[1])
        if y is None:
            y = torch.empty(self.shape[0], dtype=torch.float64, device="cuda")
        L.check(L.lib().edfa_spmv(ctx(), self.handle, dptr(x), dptr(y), alpha, beta))
        return y

    def __del__(self):
        if self._owner and self.handle and getattr(L, "_lib", None) is not None:
            try:
                L._lib.edfa_csr_destroy(self.handle)
            except Exception:   # pragma: no cover - interpreter shutdown
                pass
            self.handle = None


class DeviceSystem:
    """The 2x2 block system on the device (hx/assembly.py:135-183 layout:
    free faces first, then cells).  Keeps the host system for metadata."""

    def __init__(self, A_ff: DeviceCsr, A_fc: DeviceCsr, A_cf: DeviceCsr, A_cc: DeviceCsr,
                 rhs=None, host=None, topology_src=None):
        """``topology_src`` = (elem_to_faces, face_to_elems, face_index) of the
        grid, host arrays or CUDA tensors (default: the host system's grid)."""
        self.A_ff, self.A_fc, self.A_cf, self.A_cc = A_ff, A_fc, A_cf, A_cc
        self.host = host
        self.handle = C.c_void_p()
        L.check(L.lib().edfa_system_create(ctx(), A_ff.handle, A_fc.handle, A_cf.handle, A_cc.handle,
                                            C.byref(self.handle)))
        self._rhs = None if rhs is None else as_device_vector(rhs, self.n_unknowns)
        self._src = {}
        grid = getattr(host, "grid", None)
        self.topology = None
        if grid is not None and all(hasattr(grid, a) for a in ("nx", "ny", "nz")) \
                and grid.nx * grid.ny * grid.nz == self.n_cells:
            self.set_grid(grid.nx, grid.ny, grid.nz)
        if topology_src is not None:
            self.topology = device_topology(*topology_src)
        elif grid is not None and hasattr(host, "face_index") and hasattr(grid, "face_to_elems"):
            self.topology = device_topology(grid.elem_to_faces, grid.face_to_elems, host.face_index)

    def set_grid(self, nx: int, ny: int, nz: int) -> None:
        """Declare cells as the natural-order cells of an nx*ny*nz box
        (enables the tile-DAG Schur solves; numerics do not depend on it)."""
        L.check(L.lib().edfa_system_set_grid(self.handle, int(nx), int(ny), int(nz)))

    @classmethod
    def from_host(cls, system) -> "DeviceSystem":
        """Upload a BlockSystem (scipy CSR blocks) -- hexflow's or this repo's."""
        if isinstance(system, DeviceSystem):
            return system
        blocks = [DeviceCsr.from_scipy(getattr(system, n)) for n in ("A_ff", "A_fc", "A_cf", "A_cc")]
        ds = cls(*blocks, rhs=_upload_rhs(system), host=system)
        ds._src = {n: id(getattr(system, n)) for n in ("A_ff", "A_fc", "A_cf", "A_cc")}
        return ds

    def updated(self, system) -> "DeviceSystem":
        """Device system for ``system`` reusing every block shared by identity
        (update_accumulation replaces A_cc only, hx/assembly.py:314-333)."""
        if isinstance(system, DeviceSystem):
            return system
        if self.host is None or any(id(getattr(system, n)) != self._src.get(n)
                                    for n in ("A_ff", "A_fc", "A_cf")):
            return DeviceSystem.from_host(system)
        A_cc = self.A_cc if id(system.A_cc) == self._src.get("A_cc") else DeviceCsr.from_scipy(system.A_cc)
        ds = DeviceSystem(self.A_ff, self.A_fc, self.A_cf, A_cc, rhs=_upload_rhs(system), host=system)
        ds._src = dict(self._src, A_cc=id(system.A_cc))
        return ds

    @property
    def n_free_faces(self) -> int:
        return self.A_ff.shape[0]

    @property
    def n_cells(self) -> int:
        return self.A_cc.shape[0]

    @property
    def n_unknowns(self) -> int:
        return self.n_free_faces + self.n_cells

    def rhs(self) -> torch.Tensor:
        if self._rhs is None:
            raise ValueError("system has no right-hand side")
        return self._rhs

    def spmv(self, x, y=None) -> torch.Tensor:
        x = as_device_vector(x, self.n_unknowns)
        if y is None:
            y = torch.empty(self.n_unknowns, dtype=torch.float64, device="cuda")
        L.check(L.lib().edfa_system_spmv(ctx(), self.handle, dptr(x), dptr(y)))
        return y

    __matmul__ = spmv

    def __del__(self):
        if getattr(self, "handle", None) and getattr(L, "_lib", None) is not None:
            try:
                L._lib.edfa_system_destroy(self.handle)
            except Exception:   # pragma: no cover
                pass
            self.handle = None


def _upload_rhs(system):
    """Device right-hand side [rhs_f; rhs_c] (hx/assembly.py:172-173) uploaded
    part by part: no concatenated host copy, DMA when the parts are page-locked."""
    if hasattr(system, "rhs_f") and hasattr(system, "rhs_c"):
        parts = [np.ascontiguousarray(np.asarray(getattr(system, n), dtype=np.float64)) for n in ("rhs_f", "rhs_c")]
        out = torch.empty(sum(p.size for p in parts), dtype=torch.float64, device="cuda")
        o = 0
        for p in parts:
            out[o:o + p.size].copy_(torch.from_numpy(p), non_blocking=True)
            o += p.size
        return out
    return system.rhs() if hasattr(system, "rhs") else None


def to_host_vector(x: torch.Tensor) -> np.ndarray:
    """Device vector -> numpy through a page-locked block of torch's caching
    host allocator (DMA at full rate; the block is reused by the next call
    once the returned array is released)."""
    h = torch.empty(x.shape, dtype=x.dtype, pin_memory=True)
    h.copy_(x, non_blocking=True)
    torch.cuda.current_stream().synchronize()
    return h.numpy()


def _upload_index(a) -> torch.Tensor:
    if isinstance(a, torch.Tensor):
        return a.to("cuda").contiguous()
    a = np.asarray(a)
    if a.dtype not in (np.int32, np.int64):
        a = a.astype(np.int64)
    return torch.from_numpy(np.ascontiguousarray(a)).to("cuda", non_blocking=True)


def device_topology(elem_to_faces, face_to_elems, face_index):
    """(elem_to_faces, neighbours, face_index) as int32 CUDA tensors -- the
    inputs of the static-pattern kernel.  The grid's own index arrays are
    uploaded as they are (int32 or int64); narrowing and the neighbour map
    (hx/grid.py:100-129) are computed on the device (edfa_grid_topology)."""
    e2f_h, f2e_h, fidx_h = (_upload_index(a) for a in (elem_to_faces, face_to_elems, face_index))
    if not (e2f_h.dtype == f2e_h.dtype == fidx_h.dtype):
        e2f_h, f2e_h, fidx_h = (t.to(torch.int64) for t in (e2f_h, f2e_h, fidx_h))
    n_cells, n_faces = int(e2f_h.shape[0]), int(fidx_h.numel())
    e2f = torch.empty((n_cells, 6), dtype=torch.int32, device="cuda")
    nbr = torch.empty((n_cells, 6), dtype=torch.int32, device="cuda")
    fidx = torch.empty(n_faces, dtype=torch.int32, device="cuda")
    L.check(L.lib().edfa_grid_topology(ctx(), n_cells, n_faces, dptr(e2f_h), dptr(f2e_h), dptr(fidx_h),
                                       e2f_h.element_size(), dptr(e2f), dptr(nbr), dptr(fidx)))
    return e2f, nbr, fidx


class SystemOperator:
    """``A_apply`` callable of the monolithic block operator on the device;
    recognised by :func:`krylov.gmres`/`bicgstab` for the fused solver path."""

    def __init__(self, system: DeviceSystem):
        self.system = system

    def __call__(self, v):
        if isinstance(v, torch.Tensor):
            return self.system.spmv(v)
        return self.system.spmv(v).cpu().numpy()


def system_operator(system) -> SystemOperator:
    return SystemOperator(system if isinstance(system, DeviceSystem) else DeviceSystem.from_host(system))


def pinned_copy(system):
    """Copy of a BlockSystem whose block arrays and right-hand side live in
    page-locked host memory, so ``DeviceSystem.from_host`` uploads them by DMA
    at full PCIe/C2C bandwidth (the staging a host application keeps between
    time steps), the grid's index arrays included."""
    import dataclasses

    def pin(a):
        t = torch.from_numpy(np.ascontiguousarray(a)).pin_memory()
        return t.numpy()

    def pin_csr(M):
        M = sp.csr_matrix(M)
        return sp.csr_matrix((pin(M.data), pin(M.indices.astype(np.int32, copy=False)),
                              pin(M.indptr.astype(np.int32, copy=False))), shape=M.shape, copy=False)

    repl = {n: pin_csr(getattr(system, n)) for n in ("A_ff", "A_fc", "A_cf", "A_cc")}
    grid = getattr(system, "grid", None)
    if grid is not None and dataclasses.is_dataclass(grid) and hasattr(grid, "face_to_elems"):
        repl["grid"] = dataclasses.replace(grid, elem_to_faces=pin(grid.elem_to_faces),
                                           face_to_elems=pin(grid.face_to_elems))
    if hasattr(system, "face_index"):
        repl["face_index"] = pin(system.face_index)
    for n in ("rhs_f", "rhs_c"):
        if hasattr(system, n):
            repl[n] = pin(getattr(system, n))
    if dataclasses.is_dataclass(system):
        return dataclasses.replace(system, **repl)
    import copy
    out = copy.copy(system)
    for k, v in repl.items():
        setattr(out, k, v)
    return out
