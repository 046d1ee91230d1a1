"""Drop-in for ``hexflow.krylov`` plus GMRES(m) on the B200 path.

``bicgstab(A_apply, P_apply, b, tol, max_it)`` keeps hx/krylov.py:40-41's
signature and semantics; ``gmres(A_apply, P_apply, b, tol, restart, max_it)``
is the right-preconditioned restarted GMRES that BASELINE.json names (absent
from the reference).

Fused path: when ``A_apply`` is a device system operator (``DeviceSystem``,
``system_operator(...)`` or a preconditioner's ``device_system``) and
``P_apply`` is ``None`` or a ``BlockLDUPreconditioner`` (or its ``apply``),
the whole solve runs in libedfa (SpMV, EDFA apply, Gram-Schmidt, updates on
the device; only scalars cross to the host).

Generic path: arbitrary callables are supported for drop-in compatibility;
vectors and all Krylov arithmetic stay on the device (libedfa BLAS-1), and
the callables receive arrays of the same kind as ``b``.
"""

from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib as L
from .device import DeviceSystem, SystemOperator, as_device_vector, ctx, dptr, to_host_vector


@dataclass
class SolveReport:
    """Iteration counts, flags, residual history, timings (hx/krylov.py:15-37)."""

    n_it: int = 0
    converged: bool = False
    breakdown: bool = False
    relres_history: list = field(default_factory=list)
    final_relres: float = math.inf
    t_stage1: float = 0.0
    t_stage2: float = 0.0
    t_solve: float = 0.0
    density: float | None = None

    @property
    def t_total(self) -> float:
        return self.t_stage2 + self.t_solve

    def history_csv(self) -> str:
        lines = ["iteration,relres"] + [f"{k},{r:.6e}" for k, r in enumerate(self.relres_history)]
        return "\n".join(lines) + "\n"


def _fused_operands(A_apply, P_apply):
    """(DeviceSystem, (stage1, stage2) | None) when the fused path applies."""
    from .precond import BlockLDUPreconditioner
    if isinstance(A_apply, SystemOperator):
        sys_ = A_apply.system
    elif isinstance(A_apply, DeviceSystem):
        sys_ = A_apply
    else:
        return None
    if P_apply is None:
        return sys_, None
    pre = getattr(P_apply, "__self__", P_apply)
    if isinstance(pre, BlockLDUPreconditioner):
        if pre.stage2 is None:
            raise RuntimeError("stage 2 has not been built; call refresh()")
        return pre.stage1.system, (pre.stage1, pre.stage2)
    return None


def _run_fused(which, ops, b, tol, restart, max_it):
    sys_, stages = ops
    host = not isinstance(b, torch.Tensor)
    bd = as_device_vector(b, sys_.n_unknowns)
    x = torch.empty_like(bd)
    rep = L.Report()
    cap = max_it + 2
    hist = np.zeros(cap)
    s1 = stages[0].handle if stages else None
    s2 = stages[1].handle if stages else None
    lib = L.lib()
    if which == "gmres":
        L.check(lib.edfa_gmres(ctx(), sys_.handle, s1, s2, dptr(bd), dptr(x), float(tol), int(restart),
                               int(max_it), C.byref(rep), hist.ctypes.data_as(C.c_void_p), cap))
    else:
        L.check(lib.edfa_bicgstab(ctx(), sys_.handle, s1, s2, dptr(bd), dptr(x), float(tol), int(max_it),
                                  C.byref(rep), hist.ctypes.data_as(C.c_void_p), cap))
    r = SolveReport(n_it=rep.n_it, converged=bool(rep.converged), breakdown=bool(rep.breakdown),
                    relres_history=hist[:min(rep.n_hist, cap)].tolist(), final_relres=rep.final_relres)
    return (to_host_vector(x) if host else x), r


class _Vec:
    """Device BLAS-1 on float64 CUDA tensors through libedfa."""

    @staticmethod
    def dot(x, y) -> float:
        out = C.c_double()
        L.check(L.lib().edfa_dot(ctx(), x.numel(), dptr(x), dptr(y), C.byref(out)))
        return out.value

    @staticmethod
    def axpby(a, x, b, y):
        L.check(L.lib().edfa_axpby(ctx(), x.numel(), float(a), dptr(x), float(b), dptr(y)))
        return y


def _wrap(fn, host):
    if fn is None:
        return lambda v: v.clone()

    def call(v):
        out = fn(v.cpu().numpy() if host else v)
        return as_device_vector(out, v.numel())
    return call


def bicgstab(A_apply, P_apply, b, tol: float = 1e-8, max_it: int = 2000):
    """Right-preconditioned Bi-CGStab (hx/krylov.py:40-115): x0 = 0, stop on
    ||s||/||b|| or ||r||/||b|| <= tol, breakdowns reported, true residual
    recomputed at the end."""
    if tol <= 0:
        raise ValueError("tol must be positive")
    ops = _fused_operands(A_apply, P_apply)
    if ops is not None:
        return _run_fused("bicgstab", ops, b, tol, 0, max_it)
    host = not isinstance(b, torch.Tensor)
    A = _wrap(A_apply, host)
    P = _wrap(P_apply, host)
    bd = as_device_vector(b)
    V = _Vec
    rep = SolveReport()
    bn = math.sqrt(V.dot(bd, bd))
    if bn == 0.0:
        rep.converged, rep.final_relres = True, 0.0
        rep.relres_history.append(0.0)
        x = torch.zeros_like(bd)
        return (x.cpu().numpy() if host else x), rep
    x = torch.zeros_like(bd)
    r = bd.clone()
    rh = r.clone()
    rho = alpha = omega = 1.0
    p = torch.zeros_like(bd)
    v = torch.zeros_like(bd)
    while rep.n_it < max_it:
        rho_new = V.dot(rh, r)
        if rho_new == 0.0:
            rep.breakdown = True
            break
        beta = (rho_new / rho) * (alpha / omega)
        rho = rho_new
        V.axpby(-omega, v, 1.0, p)          # p - omega v
        V.axpby(1.0, r, beta, p)            # r + beta (p - omega v)
        ph = P(p)
        v = A(ph)
        den = V.dot(rh, v)
        if den == 0.0:
            rep.breakdown = True
            break
        alpha = rho / den
        s = V.axpby(-alpha, v, 1.0, r.clone())
        rep.n_it += 1
        sn = math.sqrt(V.dot(s, s))
        if sn / bn <= tol:
            V.axpby(alpha, ph, 1.0, x)
            rep.relres_history.append(sn / bn)
            rep.converged = True
            break
        sh = P(s)
        t = A(sh)
        tt = V.dot(t, t)
        if tt == 0.0:
            rep.breakdown = True
            break
        omega = V.dot(t, s) / tt
        V.axpby(alpha, ph, 1.0, x)
        V.axpby(omega, sh, 1.0, x)
        r = V.axpby(-omega, t, 1.0, s.clone())
        rr = math.sqrt(V.dot(r, r)) / bn
        rep.relres_history.append(rr)
        if rr <= tol:
            rep.converged = True
            break
        if omega == 0.0:
            rep.breakdown = True
            break
    if not rep.relres_history:
        rep.relres_history.append(math.sqrt(V.dot(r, r)) / bn)
    res = V.axpby(1.0, bd, -1.0, A(x))
    rep.final_relres = math.sqrt(V.dot(res, res)) / bn
    return (x.cpu().numpy() if host else x), rep


def gmres(A_apply, P_apply, b, tol: float = 1e-8, restart: int = 50, max_it: int = 2000):
    """Right-preconditioned restarted GMRES(restart), x0 = 0; converged when
    the TRUE relative residual ||b - A x|| / ||b|| <= tol."""
    if tol <= 0:
        raise ValueError("tol must be positive")
    if not 1 <= restart <= 62:
        raise ValueError("restart must be in [1, 62]")
    ops = _fused_operands(A_apply, P_apply)
    if ops is not None:
        return _run_fused("gmres", ops, b, tol, restart, max_it)
    host = not isinstance(b, torch.Tensor)
    A = _wrap(A_apply, host)
    P = _wrap(P_apply, host)
    bd = as_device_vector(b)
    n = bd.numel()
    Vb = _Vec
    rep = SolveReport()
    bn = math.sqrt(Vb.dot(bd, bd))
    if bn == 0.0:
        rep.converged, rep.final_relres = True, 0.0
        rep.relres_history.append(0.0)
        x = torch.zeros_like(bd)
        return (x.cpu().numpy() if host else x), rep
    x = torch.zeros_like(bd)
    r = bd.clone()
    beta = bn
    m = restart
    while rep.n_it < max_it:
        Vs = [Vb.axpby(1.0 / beta, r, 0.0, torch.empty(n, dtype=torch.float64, device="cuda"))]
        Hh = np.zeros((m + 1, m))
        cs, sn, g = np.zeros(m), np.zeros(m), np.zeros(m + 1)
        g[0] = beta
        k, happy = 0, False
        for j in range(m):
            w = A(P(Vs[j]))
            rep.n_it += 1
            for i in range(j + 1):          # modified Gram-Schmidt
                h = Vb.dot(w, Vs[i])
                Hh[i, j] = h
                Vb.axpby(-h, Vs[i], 1.0, w)
            hn = math.sqrt(Vb.dot(w, w))
            Hh[j + 1, j] = hn
            for i in range(j):
                a, c = Hh[i, j], Hh[i + 1, j]
                Hh[i, j] = cs[i] * a + sn[i] * c
                Hh[i + 1, j] = -sn[i] * a + cs[i] * c
            den = math.hypot(Hh[j, j], Hh[j + 1, j])
            cs[j], sn[j] = (1.0, 0.0) if den == 0.0 else (Hh[j, j] / den, Hh[j + 1, j] / den)
            Hh[j, j], Hh[j + 1, j] = den, 0.0
            g[j + 1] = -sn[j] * g[j]
            g[j] = cs[j] * g[j]
            est = abs(g[j + 1]) / bn
            rep.relres_history.append(est)
            k = j + 1
            if hn == 0.0:
                happy = True
                break
            Vs.append(Vb.axpby(1.0 / hn, w, 0.0, w))
            if est <= tol or rep.n_it >= max_it:
                break
        y = np.zeros(k)
        for i in range(k - 1, -1, -1):
            y[i] = (g[i] - Hh[i, i + 1:k] @ y[i + 1:k]) / Hh[i, i] if Hh[i, i] != 0 else 0.0
        u = torch.zeros_like(bd)
        for i in range(k):
            Vb.axpby(float(y[i]), Vs[i], 1.0, u)
        Vb.axpby(1.0, P(u), 1.0, x)
        r = Vb.axpby(1.0, bd, -1.0, A(x))
        beta = math.sqrt(Vb.dot(r, r))
        if beta / bn <= tol:
            rep.converged = True
            break
        if happy or beta == 0.0:
            rep.breakdown = True
            break
    rep.final_relres = beta / bn
    return (x.cpu().numpy() if host else x), rep
