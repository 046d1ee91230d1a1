"""C-ABI surface checks that need no GPU: libedfa.so loads, exports every
function include/edfa.h declares, and the ctypes table matches the header.

No compute entry point is called here (they need a B200)."""

import ctypes
import pathlib
import re
import subprocess

import pytest

from paper_2009_13916_b200 import _lib

ROOT = pathlib.Path(__file__).resolve().parents[1]
HEADER = ROOT / "include" / "edfa.h"


def header_functions():
    text = re.sub(r"/\*.*?\*/", "", HEADER.read_text(), flags=re.S)
    return sorted(set(re.findall(r"^\s*(?:int|int64_t|const char\*)\s+(edfa_\w+)\s*\(", text, flags=re.M)))


def test_header_declares_entry_points():
    fns = header_functions()
    assert len(fns) >= 30
    for must in ("edfa_stage1_build", "edfa_stage2_build", "edfa_precond_apply", "edfa_gmres",
                 "edfa_bicgstab", "edfa_restricted_solve", "edfa_grow_dynamic", "edfa_system_spmv"):
        assert must in fns


def test_ctypes_table_matches_header():
    assert _lib.exported_symbols() == header_functions()


def test_library_loads_and_exports_every_symbol():
    lib = _lib.lib()                      # loads libedfa.so, binds every signature
    for name in header_functions():
        assert hasattr(lib, name), name
    assert lib.edfa_abi_version() == 1


def test_dynamic_symbol_table():
    out = subprocess.run(["nm", "-D", "--defined-only", str(_lib.LIB_PATH)], capture_output=True, text=True)
    if out.returncode != 0:
        pytest.skip("nm unavailable")
    exported = set(re.findall(r"\bT (edfa_\w+)$", out.stdout, flags=re.M))
    assert set(header_functions()) <= exported


def test_library_is_sm100a():
    out = subprocess.run(["cuobjdump", "--list-elf", str(_lib.LIB_PATH)], capture_output=True, text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    assert "sm_100a" in out.stdout


def test_status_codes_map_to_reference_exceptions():
    lib = _lib.lib()
    # NULL handles are rejected with a value error before any CUDA call
    with pytest.raises(ValueError):
        _lib.check(lib.edfa_ctx_create(0, None, None))
    assert "NULL" in lib.edfa_last_error().decode()
    from paper_2009_13916_b200.errors import FactorizationError
    with pytest.raises(FactorizationError):
        _lib.check(_lib.ERR_FACTORIZATION)
    with pytest.raises(RuntimeError):
        _lib.check(_lib.ERR_STATE)
    with pytest.raises(NotImplementedError):
        _lib.check(_lib.ERR_UNSUPPORTED)


def test_csr_info_rejects_null():
    lib = _lib.lib()
    n = ctypes.c_int32()
    st = lib.edfa_csr_info(None, ctypes.byref(n), ctypes.byref(n), None)
    assert st == _lib.ERR_VALUE


def test_struct_layouts_match_header(tmp_path):
    """ctypes mirrors of the header's structs have the C sizes and offsets."""
    import shutil
    if shutil.which("gcc") is None:
        pytest.skip("gcc unavailable")
    structs = {"edfa_hex_grid": _lib.HexGridDesc, "edfa_assembly_in": _lib.AssemblyIn,
               "edfa_assembly_out": _lib.AssemblyOut, "edfa_report": _lib.Report,
               "edfa_stage1_info": _lib.Stage1Info, "edfa_stage2_info": _lib.Stage2Info,
               "edfa_dynamic": _lib.Dynamic}
    lines = ['#include <stdio.h>', '#include <stddef.h>', f'#include "{HEADER}"', "int main(void) {"]
    for cname, cls in structs.items():
        lines.append(f'printf("{cname} %zu\\n", sizeof({cname}));')
        for fname, _ in cls._fields_:
            lines.append(f'printf("{cname}.{fname} %zu\\n", offsetof({cname}, {fname}));')
    lines.append("return 0; }")
    src = tmp_path / "layout.c"
    src.write_text("\n".join(lines))
    exe = tmp_path / "layout"
    subprocess.run(["gcc", "-o", str(exe), str(src)], check=True)
    got = dict(line.rsplit(" ", 1) for line in subprocess.run([str(exe)], capture_output=True, text=True,
                                                                check=True).stdout.splitlines())
    for cname, cls in structs.items():
        assert int(got[cname]) == ctypes.sizeof(cls), cname
        for fname, _ in cls._fields_:
            assert int(got[f"{cname}.{fname}"]) == getattr(cls, fname).offset, f"{cname}.{fname}"
