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


def test_setup_and_spectral_entry_points_validate_without_a_device():
    """The device-setup, assembly and spectral entry points reject bad
    arguments before touching CUDA (status IG_INVALID_ARGUMENT + message)."""
    import ctypes as C
    lib = _ffi.gpu()
    I = _ffi.IG_INVALID_ARGUMENT
    sec = (C.c_double * 3)()
    assert lib.ig_galerkin_hierarchy(None, None, 0, None, sec) == I
    assert lib.ig_factorize_blocks(None, 0, None, None, 1e-16, None, None, sec) == I
    rank = C.c_int32()
    assert lib.ig_pstrf(-1, None, None, 0.0, C.byref(rank)) == I
    out = _ffi.ig_csr()
    assert lib.ig_assemble(None, C.byref(out), None, sec) == I
    h = C.c_void_p()
    assert lib.ig_hier_build(None, None, None, None, 2, 1e-16, 0, C.byref(h), sec) == I
    assert lib.ig_operator_columns(None, 1, 0, 1, None) == I
    assert b"null" in lib.ig_last_error()
    # an assembly payload with a bad dimension
    pay = _ffi.ig_assembly()
    pay.dim = 4
    b = np.zeros(1)
    assert lib.ig_assemble(C.byref(pay), C.byref(out), b.ctypes.data_as(C.POINTER(C.c_double)), sec) == I
    assert b"dim" in lib.ig_last_error()


def test_assembly_payload_matches_the_case(c1_case):
    """igh_assembly_payload exposes the finest space and element tables the
    host row gather used (sizes and table indices consistent)."""
    import ctypes as C
    pay = _ffi.ig_assembly()
    assert _ffi.host().igh_assembly_payload(c1_case._h, C.byref(pay)) == 0
    n = c1_case.n
    assert pay.n == n and pay.dim == 2 and pay.p == 2 and pay.family == 1
    assert pay.n_elements > 0 and pay.n_tables > 0
    tab = np.ctypeslib.as_array(pay.el_table, (pay.n_elements,))
    assert tab.min() >= 0 and tab.max() < pay.n_tables
    sp = np.ctypeslib.as_array(pay.supp_ptr, (n + 1,))
    assert sp[0] == 0 and np.all(np.diff(sp) > 0)
    # b re-summed from the payload in support (element) order equals the
    # host-assembled right-hand side bit for bit (assembly.cpp: F_e scatter).
    F = np.ctypeslib.as_array(pay.F, (pay.n_tables * 9,)).reshape(pay.n_tables, 9)
    se = np.ctypeslib.as_array(pay.supp_el, (int(sp[-1]),))
    ex = np.ctypeslib.as_array(pay.el_ix, (pay.n_elements,))
    ey = np.ctypeslib.as_array(pay.el_iy, (pay.n_elements,))
    an = np.ctypeslib.as_array(pay.anchors, (n,))
    nfx = pay.nf[0]
    b = np.zeros(n)
    for a in range(n):
        ax, ay = int(an[a] % nfx), int(an[a] // nfx)
        acc = 0.0
        for e in se[sp[a]:sp[a + 1]]:
            acc = acc + float(F[tab[e], (ay - ey[e]) * 3 + (ax - ex[e])])
        b[a] = acc
    assert np.array_equal(b, c1_case.b)
