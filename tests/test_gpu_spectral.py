"""Composed spectral operators on the device:
ig_operator_columns materialises M A / S_sym A / A column by column on the GPU
(runner.cpp:84-122, spectral.cpp:28-50); dense_spectrum finishes on the host
like the reference (dgeev)."""
import numpy as np
import pytest

import oracle_ffi as orc

pytestmark = pytest.mark.gpu


def _star(grid, smoother):
    from paper_1903_10977_b200 import CaseConfig, SmootherConfig, build_case
    return build_case(CaseConfig(geometry="star(0.037, 0.011, 0.5, 0.1, 5)", dim=2, origin=(-1, -1, 0),
                                 extent=(2, 2, 1), resolution=(grid, grid, 1), family="lagrange", degree=2,
                                 levels=2, smoother=SmootherConfig(smoother)))


def test_operator_columns_bitwise(c1_case):
    """Device columns of M A and A equal the oracle's V-cycle of the oracle's
    A e_j, bit for bit."""
    import ctypes as C
    from paper_1903_10977_b200 import MgHierarchy, _ffi
    h = MgHierarchy(c1_case)
    lv = c1_case.levels_c()
    top = h.levels() - 1
    n = h.A.rows()
    try:
        js = [0, 1, n // 3, n // 2, n - 1]
        for j in js:
            for kind in (_ffi.IG_OP_A, _ffi.IG_OP_VCYCLE):
                col = np.empty(n)
                assert _ffi.gpu().ig_operator_columns(h.handle, kind, j, 1,
                                                      col.ctypes.data_as(C.POINTER(C.c_double))) == 0
                e = np.zeros(n)
                e[j] = 1.0
                ae = orc.spmv(lv, top, e, 0)
                ref = ae if kind == _ffi.IG_OP_A else orc.vcycle_at(lv, top, ae)
                assert np.array_equal(col, ref), (j, kind)
        m = np.empty((n, 4), order="F")
        assert _ffi.gpu().ig_operator_columns(h.handle, _ffi.IG_OP_VCYCLE, 10, 4,
                                              m.ctypes.data_as(C.POINTER(C.c_double))) == 0
        for c in range(4):
            e = np.zeros(n)
            e[10 + c] = 1.0
            assert np.array_equal(m[:, c], orc.vcycle_at(lv, top, orc.spmv(lv, top, e, 0)))
    finally:
        h.close()


def test_vcycle_spectrum_in_unit_interval(c1_case):
    """MgHierarchy::apply(A .) is similar to an SPD operator with spectrum in
    (0, 1] (test_multigrid.cpp:113-120 style): real eigenvalues, lambda_max <= 1."""
    from paper_1903_10977_b200 import MgHierarchy, dense_spectrum
    h = MgHierarchy(c1_case)
    try:
        sr = dense_spectrum(h, "vcycle")
        assert sr.lambda_min > 0.0 and sr.lambda_max <= 1.0 + 1e-7
        assert 1.0 <= sr.kappa < 50.0  # damped additive Schwarz (gamma = 1/max N_K): C1 needs 25 CG iterations
        sa = dense_spectrum(h, "as2")
        assert sa.lambda_min > 0.0
        sj = dense_spectrum(h, "jacobi")
        assert sj.lambda_min > 0.0 and sj.kappa > sr.kappa
    finally:
        h.close()


def test_mesh_independence_of_the_vcycle_spectrum():
    """proj/tests/test_multigrid.cpp:195-225 on the device: on the clean star
    (Lagrange p=2, multiplicative Schwarz, 2 levels) at 16 and 32 cells per
    axis, the smoother's lambda_min decays ~4x as h halves while the V-cycle's
    stays put (drift < 25 %) and its lambda_max <= 1 + 1e-7."""
    from paper_1903_10977_b200 import MgHierarchy, dense_spectrum
    ms2_min, vc_min = [], []
    for grid in (16, 32):
        h = MgHierarchy(_star(grid, "multiplicative-schwarz"))
        try:
            ms2_min.append(dense_spectrum(h, "ms2").lambda_min)
            sv = dense_spectrum(h, "vcycle")
            vc_min.append(sv.lambda_min)
            assert sv.lambda_max <= 1.0 + 1e-7
        finally:
            h.close()
    assert ms2_min[1] > 0.0
    decay = ms2_min[0] / ms2_min[1]
    assert 4.0 / 1.5 <= decay <= 4.0 * 1.5, decay
    assert abs(vc_min[1] - vc_min[0]) / vc_min[0] < 0.25


def test_dense_spectrum_limits(c1_case):
    from paper_1903_10977_b200 import MgHierarchy, TooLarge, dense_spectrum
    h = MgHierarchy(c1_case)
    try:
        with pytest.raises(TooLarge):
            dense_spectrum(h, "vcycle", dense_limit=10)
        with pytest.raises(ValueError):
            dense_spectrum(h, "ms2")  # additive hierarchy
        with pytest.raises(ValueError):
            dense_spectrum(h, "gs3")
    finally:
        h.close()
