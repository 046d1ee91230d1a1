"""EDFA block preconditioner + Krylov solves on NVIDIA B200 (sm_100a).

Drop-in for the hot path of hexflow (arxiv 2009.13916's reproduction
package): ``hexflow.precond`` and ``hexflow.krylov`` names, signatures and
error behaviour, computed by hand-written CUDA kernels in ``libedfa.so``
behind a C ABI (``include/edfa.h``).  The input producer (grid + RT0/FV
assembly) lives in ``mesh``/``assembly``/``configs``.

GPU modules are imported lazily so the host-side input producer works on
machines without CUDA.
"""

__version__ = "0.1.0"

_LAZY = {
    "BlockLDUPreconditioner": "precond", "DynamicConfig": "precond", "Stage1": "precond",
    "Stage2": "precond", "build_stage1": "precond", "build_stage2": "precond",
    "compute_density": "precond", "grow_pattern_dynamic": "precond", "patterns_for": "precond",
    "solve_restricted_row": "precond", "InnerFactorization": "precond", "FILTRATION_MODES": "precond",
    "filter_rows": "precond", "canonical": "sparse", "mm_write": "sparse", "mm_read": "sparse",
    "SolveReport": "krylov", "bicgstab": "krylov", "gmres": "krylov",
    "PatternSet": "patterns", "base_pattern": "patterns", "static_patterns": "patterns",
    "DeviceCsr": "device", "DeviceSystem": "device", "system_operator": "device", "option": "device",
    "FactorizationError": "errors", "ConvergenceError": "errors",
}

__all__ = sorted(_LAZY)


def __getattr__(name):
    mod = _LAZY.get(name)
    if mod is None:
        raise AttributeError(name)
    import importlib
    return getattr(importlib.import_module(f"{__name__}.{mod}"), name)
