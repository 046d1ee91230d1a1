"""ctypes binding of libedfa.so (include/edfa.h).

The shared library is built in-tree (``paper_2009_13916_b200/libedfa.so``) by
``__graft_entry__.build()``.  Loading fails loudly when it is missing: there
is no CPU or PyTorch fallback for any EDFA operation.
"""

from __future__ import annotations

import ctypes as C
import os
import pathlib

from .errors import FactorizationError

LIB_PATH = pathlib.Path(__file__).resolve().parent / "libedfa.so"
if os.environ.get("EDFA_LIB"):          # A/B experiments with an alternative build
    LIB_PATH = pathlib.Path(os.environ["EDFA_LIB"]).resolve()

OK, ERR_VALUE, ERR_FACTORIZATION, ERR_STATE, ERR_CUDA, ERR_UNSUPPORTED = range(6)
FILTRATION = {"none": 0, "pre": 1, "post-schur": 2, "post-product": 3}
MEM_HOST, MEM_DEVICE = 0, 1
S1_G, S1_FT, S1_H, S1_Q, S1_L, S1_F = range(6)
S2_S, S2_L, S2_U = range(3)

vp = C.c_void_p
i32 = C.c_int32
i64 = C.c_int64
f64 = C.c_double
P_i32 = C.POINTER(C.c_int32)


class Dynamic(C.Structure):
    _fields_ = [("n_add", i32), ("n_ent", i32), ("it_max", i32)]


class Stage1Info(C.Structure):
    _fields_ = [("nnz_G", i64), ("nnz_FT", i64), ("nnz_H", i64), ("nnz_Q", i64), ("nnz_L", i64),
                ("max_pattern", i32), ("pivot_shifts", i32), ("trsv_levels", i32)]


class Stage2Info(C.Structure):
    _fields_ = [("nnz_S", i64), ("nnz_L", i64), ("nnz_U", i64), ("pivot_shifts", i32),
                ("levels_L", i32), ("levels_U", i32)]


class Report(C.Structure):
    _fields_ = [("n_it", i32), ("converged", i32), ("breakdown", i32), ("n_hist", i32),
                ("final_relres", f64)]


class HexGridDesc(C.Structure):
    _fields_ = [("n_cells", i32), ("n_faces", i32), ("n_nodes", i32), ("node_coords", vp),
                ("elem_to_nodes", vp), ("elem_to_faces", vp), ("face_to_elems", vp), ("face_local", vp),
                ("face_area", vp)]


class AssemblyIn(C.Structure):
    _fields_ = [("K", vp), ("gamma", f64), ("face_bc", vp), ("face_value", vp), ("source", vp),
                ("storage", vp), ("storage_scalar", f64)]


class AssemblyOut(C.Structure):
    _fields_ = [("face_index", vp), ("rhs_f", vp), ("rhs_c_base", vp), ("elem_volume", vp),
                ("accumulation", vp), ("binv", vp), ("row_sums", vp), ("diag", vp), ("n_free", i32),
                ("bad_element", i32)]


_SIGS = {
    "edfa_abi_version": (i32, []),
    "edfa_last_error": (C.c_char_p, []),
    "edfa_ctx_create": (i32, [i32, vp, C.POINTER(vp)]),
    "edfa_ctx_set_stream": (i32, [vp, vp]),
    "edfa_ctx_sync": (i32, [vp]),
    "edfa_ctx_trim": (i32, [vp]),
    "edfa_ctx_set_option": (i32, [vp, C.c_char_p, i32]),
    "edfa_ctx_get_option": (i32, [vp, C.c_char_p, P_i32]),
    "edfa_ctx_destroy": (i32, [vp]),
    "edfa_ctx_profile": (i32, [vp, i32]),
    "edfa_ctx_profile_filter": (i32, [vp, C.c_char_p]),
    "edfa_ctx_profile_report": (i64, [vp, C.c_char_p, i64, i32]),
    "edfa_ctx_launch_count": (i64, [vp]),
    "edfa_csr_create": (i32, [vp, i32, i32, i64, vp, vp, vp, i32, C.POINTER(vp)]),
    "edfa_csr_info": (i32, [vp, P_i32, P_i32, C.POINTER(i64)]),
    "edfa_csr_export": (i32, [vp, vp, vp, vp, vp, i32]),
    "edfa_csr_destroy": (i32, [vp]),
    "edfa_system_create": (i32, [vp, vp, vp, vp, vp, C.POINTER(vp)]),
    "edfa_system_set_cc": (i32, [vp, vp, vp]),
    "edfa_system_set_grid": (i32, [vp, i32, i32, i32]),
    "edfa_system_destroy": (i32, [vp]),
    "edfa_pattern_static": (i32, [vp, i32, i32, vp, vp, vp, C.c_char, i32, C.POINTER(vp)]),
    "edfa_grid_topology": (i32, [vp, i32, i32, vp, vp, vp, i32, vp, vp, vp]),
    "edfa_stage1_build": (i32, [vp, vp, vp, C.POINTER(Dynamic), f64, i32, f64, i32, C.POINTER(vp)]),
    "edfa_stage1_info_get": (i32, [vp, C.POINTER(Stage1Info)]),
    "edfa_stage1_part": (i32, [vp, vp, i32, C.POINTER(vp)]),
    "edfa_stage1_destroy": (i32, [vp]),
    "edfa_stage2_build": (i32, [vp, vp, vp, f64, i32, f64, i32, C.POINTER(vp)]),
    "edfa_stage2_info_get": (i32, [vp, C.POINTER(Stage2Info)]),
    "edfa_stage2_part": (i32, [vp, vp, i32, C.POINTER(vp)]),
    "edfa_stage2_destroy": (i32, [vp]),
    "edfa_precond_apply": (i32, [vp, vp, vp, vp, vp, vp]),
    "edfa_inner_apply": (i32, [vp, vp, vp, i32, vp, vp]),
    "edfa_spmv": (i32, [vp, vp, vp, vp, f64, f64]),
    "edfa_system_spmv": (i32, [vp, vp, vp, vp]),
    "edfa_restricted_solve": (i32, [vp, vp, i32, vp, vp, i32, vp, vp]),
    "edfa_grow_dynamic": (i32, [vp, vp, i32, vp, vp, C.POINTER(Dynamic), i32, vp, vp, P_i32]),
    "edfa_gmres": (i32, [vp, vp, vp, vp, vp, vp, f64, i32, i32, C.POINTER(Report), vp, i32]),
    "edfa_bicgstab": (i32, [vp, vp, vp, vp, vp, vp, f64, i32, C.POINTER(Report), vp, i32]),
    "edfa_dot": (i32, [vp, i64, vp, vp, C.POINTER(f64)]),
    "edfa_axpby": (i32, [vp, i64, f64, vp, f64, vp]),
    "edfa_csr_submatrix": (i32, [vp, vp, i32, vp, vp, i32, C.POINTER(vp)]),
    "edfa_csr_sub": (i32, [vp, vp, vp, f64, C.POINTER(vp)]),
    "edfa_csr_filter": (i32, [vp, vp, f64, i32, C.POINTER(vp)]),
    "edfa_factor_ic0": (i32, [vp, vp, f64, C.POINTER(vp)]),
    "edfa_factor_ilu0": (i32, [vp, vp, f64, i32, i32, i32, C.POINTER(vp)]),
    "edfa_factor_ic": (i32, [vp, vp, f64, i32, C.POINTER(vp)]),
    "edfa_factor_ilu": (i32, [vp, vp, f64, i32, i32, i32, i32, C.POINTER(vp)]),
    "edfa_factor_info": (i32, [vp, C.POINTER(i64), P_i32, P_i32, P_i32]),
    "edfa_factor_part": (i32, [vp, vp, i32, C.POINTER(vp)]),
    "edfa_factor_solve": (i32, [vp, vp, vp, f64, vp]),
    "edfa_factor_destroy": (i32, [vp]),
    "edfa_dcgs2_dots": (i32, [vp, i64, i32, vp, i64, vp]),
    "edfa_dcgs2_coeffs": (i32, [vp, i32, i32, vp, vp, vp, vp, vp]),
    "edfa_dcgs2_update": (i32, [vp, i64, i32, vp, i64, vp]),
    "edfa_multidot": (i32, [vp, i64, i32, vp, i64, vp, vp]),
    "edfa_multiaxpy": (i32, [vp, i64, i32, vp, i64, vp, f64, vp, vp, vp]),
    "edfa_gather": (i32, [vp, i64, vp, vp, vp]),
    "edfa_spmv_rows": (i32, [vp, vp, vp, vp, vp]),
    "edfa_assemble": (i32, [vp, C.POINTER(HexGridDesc), C.POINTER(AssemblyIn), C.POINTER(AssemblyOut),
                            C.POINTER(vp), C.POINTER(vp), C.POINTER(vp), C.POINTER(vp)]),
    "edfa_update_accumulation": (i32, [vp, vp, vp, vp, vp, f64, C.POINTER(vp), vp]),
    "edfa_face_fluxes": (i32, [vp, C.POINTER(HexGridDesc), vp, vp, vp, vp, vp, vp, vp, vp]),
    "edfa_cfl": (i32, [vp, C.POINTER(HexGridDesc), vp, vp, vp, f64, f64, vp, vp, vp, C.POINTER(f64)]),
}

_lib = None


class EdfaUnsupported(NotImplementedError):
    """Option valid in the reference but not implemented on the GPU path."""


def lib():
    """Load libedfa.so once; raise (never fall back) if it is missing."""
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise RuntimeError(
                f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
                "(the EDFA path has no CPU fallback)")
        L = C.CDLL(str(LIB_PATH))
        for name, (res, args) in _SIGS.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        if L.edfa_abi_version() != 1:
            raise RuntimeError("libedfa.so ABI version mismatch")
        _lib = L
    return _lib


def check(status: int) -> None:
    if status == OK:
        return
    msg = lib().edfa_last_error().decode(errors="replace")
    if status == ERR_VALUE:
        raise ValueError(msg)
    if status == ERR_FACTORIZATION:
        raise FactorizationError(msg)
    if status == ERR_STATE:
        raise RuntimeError(msg)
    if status == ERR_UNSUPPORTED:
        raise EdfaUnsupported(msg)
    raise RuntimeError(f"libedfa CUDA failure: {msg}")


def exported_symbols():
    """Names declared in include/edfa.h (used by the ABI tests)."""
    return sorted(_SIGS)
