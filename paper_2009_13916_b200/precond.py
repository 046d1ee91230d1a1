"""Drop-in for ``hexflow.precond`` (hx/precond.py) on the B200 path.

Same names, signatures, defaults, lifecycle and error behaviour as the
reference; every numerical step runs in libedfa.so (sm_100a):

* ``build_stage1``   restricted SPD row solves for G~/F~ (static or dynamic
                     patterns), H~ = G~ A_ff F~, IC of -A_ff   (precond.py:204-261)
* ``build_stage2``   S~ = A_cc - H~ and its ILU                 (precond.py:264-271)
* ``BlockLDUPreconditioner.apply`` block-triangular factored inverse
                                                                (precond.py:311-320)

Artefacts stay on the device; ``Stage1.G/F/H``, ``Stage2.S`` and the
factors are exported to scipy CSR only when read.
"""

from __future__ import annotations

import ctypes as C
import pathlib
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib as L
from .device import DeviceCsr, DeviceSystem, as_device_vector, ctx, dptr
from .patterns import PatternSet, as_pattern_set, base_pattern, static_patterns

FILTRATION_MODES = ("none", "pre", "post-schur", "post-product")


@dataclass(frozen=True)
class DynamicConfig:
    """Knobs of the residual-driven pattern growth (hx/precond.py:38-67)."""

    n_add: int = 1
    n_ent: int = 4
    it_max: int | None = None
    tau_filt: float = 0.0
    filtration: str = "none"

    def __post_init__(self):
        if self.n_add < 1:
            raise ValueError("n_add must be >= 1")
        if self.n_ent < 0:
            raise ValueError("n_ent must be >= 0")
        if self.it_max is not None and self.it_max < 1:
            raise ValueError("it_max must be >= 1")
        if self.filtration not in FILTRATION_MODES:
            raise ValueError(f"filtration must be one of {FILTRATION_MODES}")

    @property
    def sweep_limit(self) -> int:
        return self.it_max if self.it_max is not None else max(self.n_ent, 1)

    def _c(self):
        return L.Dynamic(self.n_add, self.n_ent, self.it_max if self.it_max is not None else 0)


def _to_host_vector(v) -> np.ndarray:
    if isinstance(v, torch.Tensor):
        return v.detach().cpu().numpy()
    return np.asarray(v, dtype=float)


class InnerFactorization:
    """Device IC/ILU factors with the reference's surface (hx/sparse.py:101-131)."""

    def __init__(self, kind, owner, part_L, part_U, nnz_stored, shifts, levels):
        self.kind = kind
        # Stage1 / Stage2 keeping the handle alive.  The owner does not hold
        # this object (it is made on access), so there is no reference cycle
        # and device memory is released as soon as the stage is dropped.
        self._owner = owner
        self._parts = (part_L, part_U)
        self._nnz_stored = nnz_stored
        self.pivot_shifts = shifts
        self.levels = levels
        self._cache = owner._cache

    @property
    def nnz_stored(self) -> int:
        return self._nnz_stored

    def _export(self, which):
        key = (self.kind, which)
        if key not in self._cache:
            if self.kind == "ic" and which == 1:
                self._cache[key] = self.L.T.tocsr()
            else:
                self._cache[key] = self._owner._part(self._parts[which]).to_scipy()
        return self._cache[key]

    @property
    def L(self):
        return self._export(0)

    @property
    def U(self):
        return self._export(1)

    def apply(self, r):
        """Approximate A^{-1} r via the two level-ordered triangular solves."""
        host = not isinstance(r, torch.Tensor)
        x = as_device_vector(r)
        y = torch.empty_like(x)
        s1 = self._owner.handle if self.kind == "ic" else None
        s2 = self._owner.handle if self.kind == "ilu" else None
        L.check(L.lib().edfa_inner_apply(ctx(), s1, s2, 0 if self.kind == "ic" else 1, dptr(x), dptr(y)))
        if host:   # the caller waits anyway: surface a solve that hit its spin limit here
            L.check(L.lib().edfa_ctx_sync(ctx()))
            return y.cpu().numpy()
        return y

    __call__ = apply


class Stage1:
    """Once-per-simulation artefacts (hx/precond.py:168-176), device-resident."""

    def __init__(self, handle, system: DeviceSystem, sets: PatternSet | None):
        self.handle = handle
        self.system = system
        info = L.Stage1Info()
        L.check(L.lib().edfa_stage1_info_get(handle, C.byref(info)))
        self.info = info
        self._cache = {}
        self._sets = sets

    @property
    def face_inner(self) -> InnerFactorization:
        n = self.system.n_free_faces
        return InnerFactorization("ic", self, L.S1_L, None, 2 * self.info.nnz_L - n, self.info.pivot_shifts,
                                  self.info.trsv_levels)

    def _part(self, which) -> DeviceCsr:
        h = C.c_void_p()
        L.check(L.lib().edfa_stage1_part(ctx(), self.handle, which, C.byref(h)))
        return DeviceCsr(h, owner=False, keepalive=self)

    def _scipy(self, which):
        if which not in self._cache:
            self._cache[which] = self._part(which).to_scipy()
        return self._cache[which]

    @property
    def G(self):
        return self._scipy(L.S1_G)

    @property
    def F(self):
        return self._scipy(L.S1_F)

    @property
    def H(self):
        return self._scipy(L.S1_H)

    @property
    def pattern_sizes(self) -> np.ndarray:
        ptr, _, _ = self._part(L.S1_Q).arrays(values=False)
        return np.diff(ptr).astype(np.int64)

    @property
    def patterns(self) -> PatternSet:
        """Restriction sets actually used (final sets for the dynamic growth)."""
        return PatternSet(device=self._part(L.S1_Q), provenance="used")

    def __del__(self):
        if getattr(self, "handle", None) and getattr(L, "_lib", None) is not None:
            try:
                L._lib.edfa_stage1_destroy(self.handle)
            except Exception:   # pragma: no cover
                pass
            self.handle = None


class Stage2:
    """Per-time-step artefacts (hx/precond.py:179-184), device-resident."""

    def __init__(self, handle, stage1: Stage1):
        self.handle = handle
        self.stage1 = stage1
        info = L.Stage2Info()
        L.check(L.lib().edfa_stage2_info_get(handle, C.byref(info)))
        self.info = info
        self._cache = {}

    @property
    def schur_inner(self) -> InnerFactorization:
        n = self.stage1.system.n_cells
        i = self.info
        return InnerFactorization("ilu", self, L.S2_L, L.S2_U, i.nnz_L - n + i.nnz_U, i.pivot_shifts,
                                  (i.levels_L, i.levels_U))

    def _part(self, which) -> DeviceCsr:
        h = C.c_void_p()
        L.check(L.lib().edfa_stage2_part(ctx(), self.handle, which, C.byref(h)))
        return DeviceCsr(h, owner=False, keepalive=self)

    @property
    def S(self):
        if "S" not in self._cache:
            self._cache["S"] = self._part(L.S2_S).to_scipy()
        return self._cache["S"]

    def __del__(self):
        if getattr(self, "handle", None) and getattr(L, "_lib", None) is not None:
            try:
                L._lib.edfa_stage2_destroy(self.handle)
            except Exception:   # pragma: no cover
                pass
            self.handle = None


def _device_system(system) -> DeviceSystem:
    return system if isinstance(system, DeviceSystem) else DeviceSystem.from_host(system)


def build_stage1(system, *, patterns=None, dynamic: DynamicConfig | None = None,
                 tau_filt: float | None = None, filtration: str | None = None,
                 face_drop_tol: float = 0.0, no_fill: bool = False, n_workers: int = 1) -> Stage1:
    """Approximate decoupling factors, their product and the face-block IC
    (hx/precond.py:204-261).  ``n_workers`` is accepted for API parity; the
    per-cell fan-out is the CUDA grid, and results never depend on it."""
    if (patterns is None) == (dynamic is None):
        raise ValueError("give exactly one of patterns or dynamic")
    if filtration is None:
        filtration = dynamic.filtration if dynamic is not None else "none"
    if tau_filt is None:
        tau_filt = dynamic.tau_filt if dynamic is not None else 0.0
    if filtration not in FILTRATION_MODES:
        raise ValueError(f"filtration must be one of {FILTRATION_MODES}")
    ds = _device_system(system)
    pat = None
    if patterns is not None:
        pat = as_pattern_set(patterns, ds.n_free_faces)
        pdev = pat.device(ds.n_free_faces)
    h = C.c_void_p()
    dyn = dynamic._c() if dynamic is not None else None
    L.check(L.lib().edfa_stage1_build(ctx(), ds.handle, pdev.handle if pat is not None else None,
                                       C.byref(dyn) if dyn is not None else None, float(tau_filt),
                                       L.FILTRATION[filtration], float(face_drop_tol), int(bool(no_fill)),
                                       C.byref(h)))
    return Stage1(h, ds, pat)


def build_stage2(A_cc, stage1: Stage1, *, tau_filt: float = 0.0, filtration: str = "none",
                 schur_drop_tol: float = 0.0, no_fill: bool = False) -> Stage2:
    """S~ = A_cc - H~ and its ILU (hx/precond.py:264-271)."""
    if filtration not in FILTRATION_MODES:
        raise ValueError(f"filtration must be one of {FILTRATION_MODES}")
    cc = A_cc if isinstance(A_cc, DeviceCsr) else DeviceCsr.from_scipy(A_cc)
    h = C.c_void_p()
    L.check(L.lib().edfa_stage2_build(ctx(), cc.handle, stage1.handle, float(tau_filt), L.FILTRATION[filtration],
                                       float(schur_drop_tol), int(bool(no_fill)), C.byref(h)))
    return Stage2(h, stage1)


@dataclass
class BlockLDUPreconditioner:
    """Two-stage factored-inverse preconditioner (hx/precond.py:274-340)."""

    system: object
    stage1: Stage1
    stage2: Stage2 | None = None
    settings: dict = field(default_factory=dict)

    @classmethod
    def build(cls, system, *, patterns=None, dynamic=None, tau_filt=None, filtration=None,
              face_drop_tol=0.0, schur_drop_tol=0.0, no_fill=False, n_workers=1):
        s1 = build_stage1(system, patterns=patterns, dynamic=dynamic, tau_filt=tau_filt,
                          filtration=filtration, face_drop_tol=face_drop_tol, no_fill=no_fill,
                          n_workers=n_workers)
        if filtration is None and dynamic is not None:
            filtration = dynamic.filtration
        if tau_filt is None and dynamic is not None:
            tau_filt = dynamic.tau_filt
        pre = cls(system, s1, settings=dict(tau_filt=tau_filt or 0.0, filtration=filtration or "none",
                                             schur_drop_tol=schur_drop_tol, no_fill=no_fill))
        pre.refresh(system)
        return pre

    @property
    def device_system(self) -> DeviceSystem:
        return self.stage1.system

    def refresh(self, system) -> None:
        """Rebuild stage 2 against a (possibly updated) cell block."""
        ds = self.stage1.system.updated(system)
        self.system = system
        self.stage1.system = ds
        self.stage2 = build_stage2(ds.A_cc, self.stage1,
                                   tau_filt=self.settings.get("tau_filt", 0.0),
                                   filtration=self.settings.get("filtration", "none"),
                                   schur_drop_tol=self.settings.get("schur_drop_tol", 0.0),
                                   no_fill=self.settings.get("no_fill", False))

    def apply(self, r):
        """Factored-inverse action; G~ and F~ are not used (Remark 1)."""
        if self.stage2 is None:
            raise RuntimeError("stage 2 has not been built; call refresh()")
        ds = self.stage1.system
        host = not isinstance(r, torch.Tensor)
        x = as_device_vector(r, ds.n_unknowns)
        y = torch.empty_like(x)
        L.check(L.lib().edfa_precond_apply(ctx(), ds.handle, self.stage1.handle, self.stage2.handle,
                                            dptr(x), dptr(y)))
        if host:   # the caller waits anyway: surface a solve that hit its spin limit here
            L.check(L.lib().edfa_ctx_sync(ctx()))
            return y.cpu().numpy()
        return y

    __call__ = apply

    @property
    def density(self) -> float:
        return compute_density(self, self.system)

    def dump(self, directory) -> None:
        """Matrix Market dump of G, F, H, S (hx/precond.py:328-340)."""
        import scipy.io
        d = pathlib.Path(directory)
        d.mkdir(parents=True, exist_ok=True)
        for name, M in (("G", self.stage1.G), ("F", self.stage1.F), ("H", self.stage1.H)):
            scipy.io.mmwrite(d / f"{name}.mtx", M, precision=17)
        if self.stage2 is not None:
            scipy.io.mmwrite(d / "S.mtx", self.stage2.S, precision=17)


def compute_density(pre: BlockLDUPreconditioner, system) -> float:
    """mu of P:689-694 (hx/precond.py:343-350)."""
    if pre.stage2 is None:
        raise RuntimeError("stage 2 has not been built")
    ds = pre.stage1.system
    num = (pre.stage1.face_inner.nnz_stored + ds.A_fc.nnz + ds.A_cf.nnz
           + pre.stage2.schur_inner.nnz_stored)
    den = ds.A_ff.nnz + ds.A_fc.nnz + ds.A_cf.nnz + ds.A_cc.nnz
    return num / den


def patterns_for(system, kind: str, prototype: str = "A", grid=None) -> PatternSet:
    """Base or static pattern set in the system's reduced numbering."""
    if kind == "base":
        if isinstance(system, DeviceSystem):
            return base_pattern(system.A_cf)
        return base_pattern(system.A_cf)
    if kind == "static":
        if isinstance(system, DeviceSystem) and grid is None and system.topology is not None:
            from .patterns import static_patterns_device
            return static_patterns_device(system.topology, prototype)
        host = system.host if isinstance(system, DeviceSystem) else system
        return static_patterns(grid or host.grid, host.face_index, prototype)
    raise ValueError(f"unknown pattern kind {kind!r}")


def solve_restricted_row(A_ff, rhs, idx) -> np.ndarray:
    """Minimum-energy approximation of (-A_ff)^{-1} rhs supported on idx
    (hx/precond.py:70-82), computed by the same warp kernel as stage 1."""
    A = A_ff if isinstance(A_ff, DeviceCsr) else DeviceCsr.from_scipy(A_ff)
    n = A.shape[0]
    rhs = _to_host_vector(rhs)
    idx = np.asarray(idx, dtype=np.int64)
    out = np.zeros(n)
    if idx.size == 0:
        return out
    if idx.min() < 0 or idx.max() >= n:
        raise IndexError("row index out of range")
    nz = np.flatnonzero(rhs)
    ri = nz.astype(np.int32)
    rv = np.ascontiguousarray(rhs[nz], dtype=np.float64)
    qi = np.ascontiguousarray(idx, dtype=np.int32)
    x = np.empty(idx.size)
    L.check(L.lib().edfa_restricted_solve(ctx(), A.handle, ri.size, ri.ctypes.data_as(C.c_void_p),
                                           rv.ctypes.data_as(C.c_void_p), qi.size,
                                           qi.ctypes.data_as(C.c_void_p), x.ctypes.data_as(C.c_void_p)))
    out[idx] = x
    return out


def grow_pattern_dynamic(A_ff, rhs_idx, rhs_val, cfg: DynamicConfig, A_csc=None):
    """Residual-driven enlargement of one starting set (hx/precond.py:107-135);
    returns (idx, x) with x the restricted solution on idx."""
    A = A_ff if isinstance(A_ff, DeviceCsr) else DeviceCsr.from_scipy(A_ff)
    ri = np.ascontiguousarray(np.asarray(rhs_idx), dtype=np.int32)
    rv = np.ascontiguousarray(np.asarray(rhs_val, dtype=float))
    cap = np.unique(ri).size + cfg.n_ent
    idx = np.empty(max(cap, 1), dtype=np.int32)
    x = np.empty(max(cap, 1))
    n_out = C.c_int32()
    dyn = cfg._c()
    L.check(L.lib().edfa_grow_dynamic(ctx(), A.handle, ri.size, ri.ctypes.data_as(C.c_void_p),
                                       rv.ctypes.data_as(C.c_void_p), C.byref(dyn), cap,
                                       idx.ctypes.data_as(C.c_void_p), x.ctypes.data_as(C.c_void_p),
                                       C.byref(n_out)))
    k = n_out.value
    return idx[:k].astype(np.int64), x[:k].copy()


def filter_rows(M, tau: float, keep_diagonal: bool = True):
    """Drop row entries below tau times the row Euclidean norm; the diagonal
    survives when keep_diagonal (hx/precond.py:138-157).  tau <= 0 returns M
    itself.  Runs as libedfa's k_filter on the device; scipy input comes back
    as canonical scipy CSR, device input (DeviceCsr) stays on the device."""
    if tau <= 0:
        return M
    from .sparse import canonical
    dev = isinstance(M, DeviceCsr)
    A = M if dev else DeviceCsr.from_scipy(canonical(M))
    h = C.c_void_p()
    L.check(L.lib().edfa_csr_filter(ctx(), A.handle, float(tau), int(bool(keep_diagonal)), C.byref(h)))
    out = DeviceCsr(h)
    return out if dev else out.to_scipy()
