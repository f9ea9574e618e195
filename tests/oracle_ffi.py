"""ctypes access to the CPU oracle (oracle/liboracle.so) -- the checker the
tests compare the GPU path against.  Test infrastructure only."""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

from paper_1903_10977_b200 import _ffi

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "oracle", "liboracle.so")
SEQ, GPU_ORDER = 0, 1

_dp = C.POINTER(C.c_double)
_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB):
            subprocess.check_call(["make", "-s", "-C", os.path.join(ROOT, "oracle")])
        L = C.CDLL(LIB)
        lvp, cop = C.POINTER(_ffi.ig_level), C.POINTER(_ffi.ig_coarse)
        L.orc_dot.argtypes = [C.c_int, C.c_int64, _dp, _dp]
        L.orc_dot.restype = C.c_double
        L.orc_spmv.argtypes = [C.POINTER(_ffi.ig_csr), _dp, _dp, C.c_int]
        L.orc_spmv_t.argtypes = [C.POINTER(_ffi.ig_csr), _dp, _dp]
        L.orc_as_apply.argtypes = [lvp, C.c_int32, _dp, _dp]
        L.orc_ms_apply.argtypes = [lvp, C.c_int32, _dp, _dp, C.c_int]
        L.orc_smoother_apply.argtypes = [lvp, C.c_int32, _dp, _dp, C.c_int]
        L.orc_coarse_solve.argtypes = [cop, _dp, _dp]
        L.orc_vcycle_at.argtypes = [lvp, C.c_int32, cop, C.c_int32, _dp, _dp]
        L.orc_pcg.argtypes = [lvp, C.c_int32, cop, C.c_int, _dp, C.c_double, C.c_int32, _dp, _dp,
                              C.POINTER(C.c_int32), _dp]
        L.orc_richardson.argtypes = L.orc_pcg.argtypes
        L.orc_set_threads.argtypes = [C.c_int]
        L.orc_get_threads.restype = C.c_int
        _lib = L
    return _lib


def set_threads(n: int) -> None:
    """Oracle thread count (n <= 0: all processors); results do not depend on it."""
    lib().orc_set_threads(int(n))


def get_threads() -> int:
    return lib().orc_get_threads()


def _p(a: np.ndarray):
    return a.ctypes.data_as(_dp)


def dot(mode, a, b):
    a = np.ascontiguousarray(a, np.float64)
    b = np.ascontiguousarray(b, np.float64)
    return lib().orc_dot(mode, a.shape[0], _p(a), _p(b))


def spmv(levels, l, x, mode=0, y=None):
    """mode 0: A x; 1: y - A x; 2: R x; 3: R^T x (same modes as ig_level_spmv)."""
    lv, nl, co = levels
    x = np.ascontiguousarray(x, np.float64)
    if mode <= 1:
        m = lv[l].A
        out = np.zeros(m.n_rows) if y is None else np.array(y, np.float64)
        lib().orc_spmv(C.byref(m), _p(x), _p(out), 1 if mode == 1 else 0)
    elif mode == 2:
        m = lv[l].R
        out = np.zeros(m.n_rows)
        lib().orc_spmv(C.byref(m), _p(x), _p(out), 0)
    else:
        m = lv[l].R
        out = np.zeros(m.n_cols)
        lib().orc_spmv_t(C.byref(m), _p(x), _p(out))
    return out


def as_apply(levels, l, r):
    lv, nl, co = levels
    r = np.ascontiguousarray(r, np.float64)
    x = np.zeros_like(r)
    lib().orc_as_apply(C.byref(lv[l]), r.shape[0], _p(r), _p(x))
    return x


def smoother_apply(levels, l, r, direction=0):
    """The level's smoother (additive or multiplicative); direction 0 Forward, 1 Reverse."""
    lv, nl, co = levels
    r = np.ascontiguousarray(r, np.float64)
    x = np.zeros_like(r)
    lib().orc_smoother_apply(C.byref(lv[l]), r.shape[0], _p(r), _p(x), direction)
    return x


def coarse_solve(levels, r):
    lv, nl, co = levels
    r = np.ascontiguousarray(r, np.float64)
    x = np.zeros_like(r)
    lib().orc_coarse_solve(co, _p(r), _p(x))
    return x


def vcycle_at(levels, l, r):
    lv, nl, co = levels
    r = np.ascontiguousarray(r, np.float64)
    x = np.zeros_like(r)
    rc = lib().orc_vcycle_at(lv, nl, co, l, _p(r), _p(x))
    assert rc == 0
    return x


def richardson(levels, b, tol=1e-10, maxit=1000, mode=SEQ):
    """(status, x, residuals[:it+1], iterations, seconds)."""
    lv, nl, co = levels
    b = np.ascontiguousarray(b, np.float64)
    x = np.zeros_like(b)
    res = np.zeros(maxit + 1)
    it, sec = C.c_int32(), C.c_double()
    st = lib().orc_richardson(lv, nl, co, mode, _p(b), tol, maxit, _p(x), _p(res), C.byref(it), C.byref(sec))
    return st, x, res[:it.value + 1].copy(), it.value, sec.value


def pcg(levels, b, tol=1e-10, maxit=1000, mode=SEQ):
    """Returns (status, x, residuals, iterations, seconds)."""
    lv, nl, co = levels
    b = np.ascontiguousarray(b, np.float64)
    x = np.zeros_like(b)
    res = np.zeros(maxit + 1)
    it = C.c_int32()
    sec = C.c_double()
    st = lib().orc_pcg(lv, nl, co, mode, _p(b), tol, maxit, _p(x), _p(res), C.byref(it), C.byref(sec))
    return st, x, res[: it.value + 1].copy(), it.value, sec.value


class Synthetic:
    """A hand-built hierarchy payload (levels + coarse factor) from numpy
    arrays, for the reference's small algebraic fixtures (identity CG,
    indefinite breakdown) that do not come from a mesh."""

    def __init__(self, A_dense: np.ndarray):
        import scipy.linalg.lapack as lapack
        n = A_dense.shape[0]
        self.keep = []
        rp, ci, vv = [0], [], []
        for i in range(n):
            for j in range(n):
                if A_dense[i, j] != 0.0:
                    ci.append(j)
                    vv.append(A_dense[i, j])
            rp.append(len(ci))
        rp = np.array(rp, np.int32)
        ci = np.array(ci if ci else [0], np.int32)
        vv = np.array(vv if vv else [0.0], np.float64)
        self.keep += [rp, ci, vv]
        lv = (_ffi.ig_level * 1)()
        lv[0].A.n_rows = lv[0].A.n_cols = n
        lv[0].A.nnz = int(rp[-1])
        lv[0].A.row_ptr = rp.ctypes.data_as(C.POINTER(C.c_int32))
        lv[0].A.col_idx = ci.ctypes.data_as(C.POINTER(C.c_int32))
        lv[0].A.val = vv.ctypes.data_as(_dp)
        lv[0].smoother_kind = _ffi.IG_SMOOTHER_ADDITIVE_SCHWARZ
        # coarse = pivoted Cholesky of the (only) level, as MgHierarchy::build with levels = 1
        a = np.asfortranarray(A_dense.astype(np.float64).copy())
        tol = 1e-14 * max(0.0, float(np.max(np.diag(a))) if n else 0.0)
        piv = np.zeros(max(n, 1), np.int32)
        from paper_1903_10977_b200 import _ffi as F
        rank = F.host().igh_pstrf(n, a.ctypes.data_as(_dp), piv.ctypes.data_as(C.POINTER(C.c_int32)), tol)
        self.keep += [a, piv]
        co = _ffi.ig_coarse()
        co.n = n
        co.rank = rank
        co.L = a.ctypes.data_as(_dp)
        co.piv = piv.ctypes.data_as(C.POINTER(C.c_int32))
        self.lv, self.co = lv, co
        self.keep += [lv, co]

    def levels_c(self):
        return self.lv, 1, C.pointer(self.co)
