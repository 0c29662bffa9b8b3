"""The C-ABI library: builds for sm_100a, loads, and exports exactly what
include/srj.h declares (CPU; no CUDA call is made)."""

from __future__ import annotations

import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "srj.h")
LIB = os.path.join(ROOT, "paper_2011_06636_b200", "libsrj.so")


def declared_functions():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"^\s*(?:const\s+)?\w+\*?\s+\**(srj_\w+)\s*\(", text, flags=re.M)))


def test_header_declares_the_documented_entry_points():
    names = declared_functions()
    for must in ("srj_op_create", "srj_run_cycle", "srj_residual_sq", "srj_sweep",
                 "srj_sweep_planes", "srj_matvec", "srj_fill_uniform_rhs", "srj_last_error"):
        assert must in names


def test_library_exports_every_declared_symbol():
    if not os.path.exists(LIB):
        pytest.skip("libsrj.so not built")
    L = ctypes.CDLL(LIB)
    for name in declared_functions():
        assert hasattr(L, name), name
    from paper_2011_06636_b200 import _lib
    assert set(_lib.EXPORTED_SYMBOLS) == set(declared_functions())


def test_library_is_sm100a_code():
    if not os.path.exists(LIB):
        pytest.skip("libsrj.so not built")
    out = subprocess.run(["cuobjdump", "--list-elf", LIB], capture_output=True, text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    assert "sm_100a" in out.stdout


def test_abi_version_and_error_string_without_gpu():
    if not os.path.exists(LIB):
        pytest.skip("libsrj.so not built")
    from paper_2011_06636_b200 import _lib
    L = _lib.load()
    assert L.srj_abi_version() == _lib.ABI_VERSION
    # argument validation happens before any CUDA call
    rc = L.srj_op_create(None, None)
    assert rc == _lib.SRJ_BAD_ARGUMENT
    assert b"null" in L.srj_last_error()
    desc = _lib.OpDesc(family=99, device=0, nx=4, ny=1, nz=1, dx2=25.0)
    h = ctypes.c_void_p()
    assert L.srj_op_create(ctypes.byref(desc), ctypes.byref(h)) == _lib.SRJ_BAD_ARGUMENT
    assert b"family" in L.srj_last_error()
    assert L.srj_op_planes(None) == -1


def test_kernels_use_tma_and_no_fma_in_the_stencil():
    """SASS evidence: the tiled kernels issue TMA loads (UTMALDG) and the
    temporally blocked kernel's arithmetic is separately rounded DADD/DMUL."""
    if not os.path.exists(LIB):
        pytest.skip("libsrj.so not built")
    out = subprocess.run(["cuobjdump", "-sass", LIB], capture_output=True, text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    sass = out.stdout
    assert "UTMALDG.2D" in sass and "UTMALDG.3D" in sass
    assert "DADD" in sass and "DMUL" in sass


def test_missing_library_fails_loudly(tmp_path, monkeypatch):
    """No CPU fallback: without libsrj.so the operator layer raises."""
    from paper_2011_06636_b200 import _lib
    monkeypatch.setattr(_lib, "_lib", None)
    with pytest.raises(_lib.SrjLibraryError, match="no CPU fallback"):
        _lib.load(str(tmp_path / "libsrj.so"))
