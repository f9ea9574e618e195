"""Multiplicative (colored) Schwarz on the device: every piece bit-identical
to the oracle's restatement of smoothers.cpp:186-208 (Forward in the
pre-smoother, Reverse in the post-smoother of vcycle_at), and the whole
MS-preconditioned PCG bit-identical to the GPU-order oracle."""
import numpy as np
import pytest

import oracle_ffi as orc
from conftest import rng_vec

pytestmark = pytest.mark.gpu

UNIT = dict(origin=(-1, -1, 0), extent=(2, 2, 1))


def _cases():
    from paper_1903_10977_b200 import CaseConfig, SmootherConfig, configs
    ms = SmootherConfig("multiplicative-schwarz")
    c1 = configs.c1()
    c1.smoother = ms
    return {
        "c1": c1,
        "star-lagrange": CaseConfig(geometry="star(0.037, 0.011, 0.5, 0.1, 5)", resolution=(16, 16, 1),
                                    family="lagrange", degree=2, levels=3, smoother=ms, **UNIT),
        "thb-refined": CaseConfig(geometry="star(0.037, 0.011, 0.5, 0.1, 5)", resolution=(16, 16, 1), family="thb",
                                  degree=2, levels=3, refine_boxes=[(-0.24, -0.24, 0.24, 0.24)], smoother=ms, **UNIT),
        "3d": CaseConfig(geometry=configs.c4_geometry(1), dim=3, resolution=(16, 16, 16), degree=2, levels=3,
                         quad_depth=2, origin=(0, 0, 0), extent=(1, 1, 1), dirichlet_box_sides=False, smoother=ms),
    }


@pytest.fixture(scope="module", params=["c1", "star-lagrange", "thb-refined", "3d"])
def ms_hier(request):
    """The device sweep (per-colour block solves + residual updates)."""
    from paper_1903_10977_b200 import MgHierarchy, build_case
    case = build_case(_cases()[request.param])
    h = MgHierarchy(case)
    yield h
    h.close()


def test_smoother_forward_bitwise(ms_hier):
    h = ms_hier
    lv = h.case.levels_c()
    for l in range(1, h.levels()):
        r = rng_vec(31 + l, h._n[l])
        assert np.array_equal(h.smoother_apply(l, r), orc.smoother_apply(lv, l, r, 0))


def test_vcycle_bitwise(ms_hier):
    h = ms_hier
    lv = h.case.levels_c()
    for l in range(h.levels()):
        r = rng_vec(41 + l, h._n[l])
        assert np.array_equal(h.vcycle_at(l, r), orc.vcycle_at(lv, l, r))


def test_pcg_bitwise(ms_hier):
    from paper_1903_10977_b200 import pcg
    h = ms_hier
    lv = h.case.levels_c()
    b = h.case.b
    x, rep = pcg(h.A, b, h, tol=1e-8, maxit=1000)
    st, xo, ro, it, _ = orc.pcg(lv, b, tol=1e-8, maxit=1000, mode=orc.GPU_ORDER)
    assert st == 0 and rep.converged and rep.iterations == it
    assert np.array_equal(np.array(rep.residuals), ro)
    assert np.array_equal(x, xo)


def test_smoother_reverse_and_symmetric_bitwise(ms_hier):
    """Smoother::apply(r, Reverse) and apply_symmetric (smoothers.cpp:211-214)
    on the device against the oracle's pieces."""
    h = ms_hier
    lv = h.case.levels_c()
    for l in range(1, h.levels()):
        r = rng_vec(61 + l, h._n[l])
        assert np.array_equal(h.smoother_apply(l, r, 1), orc.smoother_apply(lv, l, r, 1))
        x1 = orc.smoother_apply(lv, l, r, 0)
        res = orc.spmv(lv, l, x1, 1, r.copy())
        want = x1 + orc.smoother_apply(lv, l, res, 1)
        assert np.array_equal(h.smoother_apply_symmetric(l, r), want)
