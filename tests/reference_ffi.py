"""ctypes access to oracle/_ref/libimmergrid_ref.so: the reference's own
solvers.cpp / multigrid.cpp / smoothers.cpp compiled unmodified against the
Eigen / LAPACKE stand-in (oracle/ref_shim, oracle/ref_glue.cpp; built by
`make -C oracle ref` where /root/reference exists).  Test infrastructure
only: the checker the oracle is pinned against."""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

from paper_1903_10977_b200 import _ffi

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "oracle", "_ref", "libimmergrid_ref.so")

_dp = C.POINTER(C.c_double)
_ip = C.POINTER(C.c_int32)
_lib = None


def available() -> bool:
    return os.path.exists(LIB)


def lib():
    global _lib
    if _lib is None:
        L = C.CDLL(LIB)
        lvp, cop = C.POINTER(_ffi.ig_level), C.POINTER(_ffi.ig_coarse)
        L.ref_hier_create.argtypes = [lvp, C.c_int32, cop]
        L.ref_hier_create.restype = C.c_void_p
        L.ref_hier_free.argtypes = [C.c_void_p]
        L.ref_coarse_rank.argtypes = [C.c_void_p]
        L.ref_block_factor.argtypes = [C.c_void_p, C.c_int32, C.c_int32, _dp]
        L.ref_vcycle_at.argtypes = [C.c_void_p, C.c_int32, _dp, C.c_int64, _dp]
        L.ref_coarse_solve.argtypes = [C.c_void_p, _dp, C.c_int64, _dp]
        L.ref_smoother_apply.argtypes = [C.c_void_p, C.c_int32, _dp, C.c_int64, _dp, C.c_int32]
        L.ref_smoother_apply_symmetric.argtypes = [C.c_void_p, C.c_int32, _dp, C.c_int64, _dp]
        L.ref_pcg.argtypes = [C.c_void_p, _dp, C.c_int64, C.c_double, C.c_int32, _dp, _dp, _ip, _ip]
        L.ref_richardson.argtypes = L.ref_pcg.argtypes
        L.ref_factorize_blocks.argtypes = [C.POINTER(_ffi.ig_csr), C.c_int32, _ip, _ip, C.c_double, _ip, _ip,
                                           C.POINTER(C.c_int64), _dp]
        L.ref_coarse_factor.argtypes = [C.POINTER(_ffi.ig_csr), _dp, _ip]
        _lib = L
    return _lib


def _p(a):
    return a.ctypes.data_as(_dp)


class RefHierarchy:
    """The payload (levels_c() of a Case or of oracle_ffi.Synthetic) as the
    reference's immergrid::MgHierarchy."""

    def __init__(self, levels):
        self.lv, self.nl, self.co = levels
        self.h = lib().ref_hier_create(self.lv, self.nl, self.co)
        assert self.h, "ref_hier_create failed"

    def close(self):
        if self.h:
            lib().ref_hier_free(self.h)
            self.h = None

    def __del__(self):
        self.close()

    def n(self, l):
        return self.lv[l].A.n_rows

    def _call(self, fn, r, *args):
        r = np.ascontiguousarray(r, np.float64)
        x = np.zeros_like(r)
        rc = fn(r, x, *args)
        return rc, x

    def vcycle_at(self, l, r):
        r = np.ascontiguousarray(r, np.float64)
        x = np.zeros_like(r)
        rc = lib().ref_vcycle_at(self.h, l, _p(r), r.shape[0], _p(x))
        return rc, x

    def coarse_solve(self, r):
        r = np.ascontiguousarray(r, np.float64)
        x = np.zeros_like(r)
        assert lib().ref_coarse_solve(self.h, _p(r), r.shape[0], _p(x)) == 0
        return x

    def smoother_apply(self, l, r, direction=0):
        r = np.ascontiguousarray(r, np.float64)
        x = np.zeros_like(r)
        assert lib().ref_smoother_apply(self.h, l, _p(r), r.shape[0], _p(x), direction) == 0
        return x

    def smoother_apply_symmetric(self, l, r):
        r = np.ascontiguousarray(r, np.float64)
        x = np.zeros_like(r)
        assert lib().ref_smoother_apply_symmetric(self.h, l, _p(r), r.shape[0], _p(x)) == 0
        return x

    def _solve(self, fn, b, tol, maxit):
        b = np.ascontiguousarray(b, np.float64)
        x = np.zeros_like(b)
        res = np.zeros(maxit + 2)
        it, nres = C.c_int32(), C.c_int32()
        st = fn(self.h, _p(b), b.shape[0], tol, maxit, _p(x), _p(res), C.byref(it), C.byref(nres))
        return st, x, res[:nres.value].copy(), it.value

    def pcg(self, b, tol=1e-10, maxit=1000):
        """(status, x, residuals, iterations) of the reference's pcg with precond = MgHierarchy::apply."""
        return self._solve(lib().ref_pcg, b, tol, maxit)

    def richardson(self, b, tol=1e-10, maxit=1000):
        return self._solve(lib().ref_richardson, b, tol, maxit)

    def block_factor(self, l, b, s):
        out = np.zeros(s * s)
        assert lib().ref_block_factor(self.h, l, b, _p(out)) == s
        return out


def factorize_blocks(A_c, ptr, dofs, filter_ratio):
    """The reference's factorize_blocks on a pre-filter layout -> (status, ptr, dofs, fac_ptr, fac)."""
    ptr = np.ascontiguousarray(ptr, np.int32)
    dofs = np.ascontiguousarray(dofs, np.int32)
    nb = ptr.shape[0] - 1
    sizes = np.diff(ptr).astype(np.int64)
    optr = np.zeros(nb + 1, np.int32)
    odofs = np.zeros(max(1, dofs.shape[0]), np.int32)
    fptr = np.zeros(nb + 1, np.int64)
    fac = np.zeros(max(1, int((sizes * sizes).sum())))
    st = lib().ref_factorize_blocks(C.byref(A_c), nb, ptr.ctypes.data_as(_ip), dofs.ctypes.data_as(_ip), filter_ratio,
                                    optr.ctypes.data_as(_ip), odofs.ctypes.data_as(_ip),
                                    fptr.ctypes.data_as(C.POINTER(C.c_int64)), _p(fac))
    return st, optr, odofs[:optr[-1]], fptr, fac[:fptr[-1]]


def coarse_factor(A_c):
    n = A_c.n_rows
    L = np.zeros(max(1, n * n))
    piv = np.zeros(max(1, n), np.int32)
    rank = lib().ref_coarse_factor(C.byref(A_c), _p(L), piv.ctypes.data_as(_ip))
    return rank, L[:n * n], piv[:n]
