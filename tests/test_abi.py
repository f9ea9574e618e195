"""The C-ABI libraries load without a GPU and export every symbol the headers
declare; the Python mirror refuses CPU fallbacks.  CPU only."""
import os
import re

import numpy as np
import pytest

from paper_1903_10977_b200 import _ffi

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared(header):
    text = open(os.path.join(ROOT, "include", header)).read()
    return sorted(set(re.findall(r"^\s*(?:int|void|const char|void \*|int32_t)\s*\*?\s*(ig[h]?_\w+)\s*\(",
                                 text, re.M)))


def test_gpu_library_exports_every_declared_symbol():
    lib = _ffi.gpu()
    names = declared("ig_gpu.h")
    assert len(names) >= 15
    missing = [s for s in names if not hasattr(lib, s)]
    assert not missing, missing
    assert set(_ffi.GPU_SYMBOLS) <= set(names)


def test_host_library_exports_every_declared_symbol():
    lib = _ffi.host()
    names = declared("ig_host.h")
    assert len(names) >= 10
    missing = [s for s in names if not hasattr(lib, s)]
    assert not missing, missing


def test_gpu_library_is_sm100a_native():
    import subprocess
    out = subprocess.run(["cuobjdump", "--list-elf", os.path.join(ROOT, "paper_1903_10977_b200", "libig_gpu.so")],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_pcg_rejects_a_non_device_preconditioner(c1_case):
    from paper_1903_10977_b200 import pcg
    with pytest.raises(TypeError):
        pcg(c1_case.A, c1_case.b, lambda r: r)


def test_create_rejects_bad_payload_without_a_device():
    """Argument validation happens before any CUDA call."""
    import ctypes as C
    lib = _ffi.gpu()
    h = C.c_void_p()
    assert lib.ig_hier_create(None, 0, None, C.byref(h)) == _ffi.IG_INVALID_ARGUMENT
    assert b"levels" in lib.ig_last_error()
