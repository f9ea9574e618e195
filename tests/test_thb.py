"""THB host setup (configs[4], C5): hierarchical mesh, truncated hierarchical
B-spline space, THB restriction and the Galerkin hierarchy the solve phase
consumes.  CPU only; the GPU parity of C5 lives in test_gpu_configs.py.

Pins: the reference's MBB space size (proj/tests/test_runner.cpp:438-445),
THB == B-spline on an unrefined mesh (truncation is the identity there,
proj/src/basis.cpp THB branch), and partition of unity carried through the
restriction (proj/tests/test_basis.cpp:92-110 states it for the basis; a
nested hierarchy then forces unit column sums of R).
"""
import ctypes as C

import numpy as np
import pytest

import oracle_ffi as orc
from paper_1903_10977_b200 import CaseConfig, _ffi, build_case, configs

UNIT = dict(origin=(-1, -1, 0), extent=(2, 2, 1))
STAR = "star(0.037, 0.011, 0.5, 0.1, 5)"


def n_dofs(cfg):
    c = cfg.to_c()
    eta, cut, n = C.c_double(), C.c_int64(), C.c_int32()
    assert _ffi.host().igh_eta(C.byref(c), C.byref(eta), C.byref(cut), C.byref(n)) == 0
    return n.value


def test_mbb_space_size():
    """proj/cases/mbb.toml geometry/mesh/refine boxes; the reference counts
    2 components (4354), the scalar space here is half of it."""
    cfg = CaseConfig(geometry="complement(union(disc(0.8, 0.45, 0.25), disc(1.8, 0.55, 0.3), "
                              "disc(2.55, 0.35, 0.18)))",
                     origin=(0, 0, 0), extent=(3, 1, 1), resolution=(60, 20, 1), family="thb", degree=2,
                     refine_boxes=[(0.0, 0.55, 0.9, 1.0), (0.0, 0.8, 0.45, 1.0)])
    assert 2 * n_dofs(cfg) == 4354


@pytest.mark.parametrize("geometry", ["constant(1)", STAR])
def test_thb_equals_bspline_unrefined(geometry):
    kw = dict(geometry=geometry, resolution=(16, 16, 1), degree=2, levels=3, **UNIT)
    a = build_case(CaseConfig(family="bspline", **kw))
    t = build_case(CaseConfig(family="thb", **kw))
    assert a.level_dofs() == t.level_dofs()
    for l in range(3):
        A1, A2 = a.level_A(l).to_scipy(), t.level_A(l).to_scipy()
        assert abs(A1 - A2).max() <= 1e-13 * abs(A1).max()
    for l in range(1, 3):
        R1, R2 = a.level_R(l).to_scipy(), t.level_R(l).to_scipy()
        assert abs(R1 - R2).max() <= 1e-13


def _refined(geometry="constant(1)", levels=2):
    """proj/tests/test_basis.cpp:35-39: base 16^2, box |x|,|y| <= 0.24 refined."""
    return build_case(CaseConfig(geometry=geometry, resolution=(16, 16, 1), family="thb", degree=2,
                                 levels=levels, refine_boxes=[(-0.24, -0.24, 0.24, 0.24)], **UNIT))


def test_refined_restriction_partition_of_unity():
    case = _refined(levels=3)
    n = case.level_dofs()
    assert n[-1] > 324  # the refined block adds fine functions on top of the 18^2 base
    for l in range(1, case.n_levels):
        R = case.level_R(l).to_scipy()
        assert R.shape == (n[l - 1], n[l])
        assert np.abs(np.asarray(R.sum(axis=0)).ravel() - 1.0).max() <= 1e-12
        assert R.min() >= -1e-14  # THB restriction coefficients are nonnegative


def test_refined_galerkin_and_spd():
    case = _refined(STAR, levels=3)
    for l in range(1, case.n_levels):
        R = case.level_R(l).to_scipy()
        Af, Ac = case.level_A(l).to_scipy(), case.level_A(l - 1).to_scipy()
        G = (R @ Af @ R.T).tocsr()
        assert abs(G - Ac).max() <= 1e-12 * abs(Ac).max()
    A = case.A.to_scipy().toarray()
    assert np.allclose(A, A.T, rtol=0, atol=1e-14 * abs(A).max())
    assert np.linalg.eigvalsh(A).min() > 0


def test_refined_pcg_converges():
    case = _refined(STAR, levels=3)
    st, x, res, it, _ = orc.pcg(case.levels_c(), case.b, tol=1e-10, maxit=200, mode=orc.SEQ)
    assert st == 0 and it < 60
    A = case.A.to_scipy()
    assert np.linalg.norm(case.b - A @ x) <= 1e-9 * np.linalg.norm(case.b)


def test_c5_full_size_hierarchy():
    """configs[4]: base 128^2, two refinement passes near the circle, 6 levels."""
    case = build_case(configs.c5())
    assert case.level_dofs() == [164, 379, 972, 3080, 10810, 40211]
    assert case.A.nnz == 1004619
    assert case.info.coarse_rank == 155
    assert max(case.info.max_nk[l] for l in range(case.n_levels)) == 17
    st, x, res, it, _ = orc.pcg(case.levels_c(), case.b, tol=1e-8, maxit=1000, mode=orc.SEQ)
    assert st == 0 and it == 37
