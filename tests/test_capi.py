"""CPU: the C-ABI library loads, exports every symbol include/*.h declares,
and the ctypes argument structs match the C layout (checked with gcc).
No compute calls (no GPU here)."""

import ctypes as C
import os
import re
import subprocess
import tempfile

import pytest

from conftest import REPO

HEADER = os.path.join(REPO, "include", "tensortrack_b200.h")


def declared_symbols():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(tt_[a-z0-9_]+)\s*\(", text)))


def test_library_loads_and_exports_every_declared_symbol():
    from paper_1609_04104_b200 import _lib

    lib = _lib.load()
    syms = declared_symbols()
    assert len(syms) >= 15
    for s in syms:
        assert hasattr(lib, s), f"missing export {s}"
        assert s in _lib.SIGNATURES, f"no ctypes signature for {s}"
    assert lib.tt_version().decode().startswith("tensortrack_b200")


def test_pure_host_queries():
    from paper_1609_04104_b200 import _lib

    lib = _lib.load()
    cl = C.c_int(0)
    sm = C.c_size_t(0)
    assert lib.tt_rows_plan(256, 256, 20, 64, 1, C.byref(cl), C.byref(sm)) == 0
    assert cl.value in (1, 2, 4, 8, 16) and 0 < sm.value <= 227 * 1024
    assert lib.tt_rows_scratch_bytes(1, 256, 256, 20, 64, cl.value) > 0
    # invalid plan -> TT_EINVAL, message recorded
    assert lib.tt_rows_plan(0, 256, 20, 64, 1, C.byref(cl), C.byref(sm)) == _lib.TT_EINVAL
    assert b"bad shape" in lib.tt_last_error()
    cl = C.c_int(3)
    assert lib.tt_rows_plan(256, 256, 20, 64, 1, C.byref(cl), C.byref(sm)) == _lib.TT_EINVAL


def test_error_codes_map_to_reference_exceptions():
    from paper_1609_04104_b200 import _lib

    with pytest.raises(ValueError):
        _lib.check(_lib.TT_EINVAL)
    with pytest.raises(TypeError):
        _lib.check(_lib.TT_EUNSUPPORTED)
    with pytest.raises(_lib.NumericalError):
        _lib.check(_lib.TT_ENONFINITE)
    with pytest.raises(RuntimeError):
        _lib.check(_lib.TT_ECUDA)
    with pytest.raises(ValueError):
        _lib.raise_status(_lib.TT_ST_DUPROW, "x")
    with pytest.raises(_lib.NumericalError):
        _lib.raise_status(_lib.TT_ST_NONFINITE, "x")


@pytest.mark.parametrize("struct,cname", [("RowsArgs", "tt_rows_args"), ("EntriesArgs", "tt_entries_args"),
                                          ("PatchesArgs", "tt_patches_args")])
def test_ctypes_struct_layout_matches_c(struct, cname):
    from paper_1609_04104_b200 import _lib

    S = getattr(_lib, struct)
    fields = [f[0] for f in S._fields_]
    src = ["#include <stdio.h>", "#include <stddef.h>", f'#include "{HEADER}"', "int main(void){",
           f'printf("%zu\\n", sizeof({cname}));']
    src += [f'printf("%zu\\n", offsetof({cname}, {f}));' for f in fields]
    src.append("return 0;}")
    with tempfile.TemporaryDirectory() as d:
        c = os.path.join(d, "l.c")
        open(c, "w").write("\n".join(src))
        exe = os.path.join(d, "l")
        subprocess.run(["gcc", c, "-o", exe], check=True)
        vals = [int(v) for v in subprocess.run([exe], capture_output=True, text=True, check=True).stdout.split()]
    assert vals[0] == C.sizeof(S)
    for f, off in zip(fields, vals[1:]):
        assert getattr(S, f).offset == off, f
