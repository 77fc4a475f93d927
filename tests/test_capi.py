"""The C-ABI library (CPU-side checks): it loads, exports every symbol include/rkb200.h
declares, reports its version, maps argument errors to RK_EINVAL, and -- with no GPU --
refuses to run instead of falling back to the CPU."""

import ctypes
import re
from pathlib import Path

import numpy as np
import pytest

from paper_1810_01051_b200 import _lib

HEADER = Path(__file__).resolve().parent.parent / "include" / "rkb200.h"


def declared_functions():
    text = HEADER.read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(rk_[a-z_0-9]+)\s*\(", text)))


def test_header_lists_match():
    assert declared_functions() == sorted(_lib.EXPORTS)


def test_library_exports_every_symbol():
    L = _lib.lib()
    for name in declared_functions():
        assert hasattr(L, name), name


def test_version_and_error_string():
    L = _lib.lib()
    assert L.rk_version().decode().startswith("rkb200 ")
    assert "sm_100a" in L.rk_version().decode()
    assert isinstance(L.rk_last_error(), bytes)


def test_null_context_is_einval():
    L = _lib.lib()
    mt = ctypes.c_uint64()
    rc = L.rk_scan(None, None, 0, b"ab", 2, 292, 0, 0, None, 0, ctypes.byref(mt),
                   ctypes.byref(mt), ctypes.byref(mt), None)
    assert rc == _lib.RK_EINVAL
    assert b"context" in L.rk_last_error()
    with pytest.raises(ValueError):
        _lib.check(rc)


def test_no_gpu_means_no_scan():
    L = _lib.lib()
    if L.rk_device_count() > 0:
        pytest.skip("a GPU is visible; covered by the gpu tests")
    h = ctypes.c_void_p()
    rc = L.rk_ctx_create(0, ctypes.byref(h))
    assert rc == _lib.RK_ECUDA and not h.value
    import paper_1810_01051_b200 as rk

    with pytest.raises(RuntimeError):
        rk.search_sequential(b"abab", b"ab")


def test_library_is_sm100a_only():
    """cuobjdump lists exactly one ELF target, sm_100a (no PTX or other-arch fallback)."""
    import shutil
    import subprocess

    exe = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    if not Path(exe).exists():
        pytest.skip("cuobjdump not available")
    out = subprocess.run([exe, "--list-elf", str(_lib.LIB_PATH)], capture_output=True,
                         text=True).stdout
    archs = set(re.findall(r"sm_\d+a?", out))
    assert archs == {"sm_100a"}, out
    ptx = subprocess.run([exe, "--list-ptx", str(_lib.LIB_PATH)], capture_output=True,
                         text=True).stdout
    assert "ptx" not in ptx.lower() or ptx.strip() == ""


def test_host_buffers_roundtrip_types():
    # argtypes accept numpy pointers as plain integers
    a = np.arange(4, dtype=np.int64)
    assert a.ctypes.data != 0
