"""Preconditioned Richardson (solvers.cpp:73-120).
CPU: the oracle restatement against the reference's own tests
(proj/tests/test_solvers.cpp:109-151): the damped two-level cycle contracts
at 1 - lambda_min (25..60 iterations, last ratios in (0.5, 0.6)); the
undamped additive cycle diverges (Diverged after 10 growths).  GPU: the
device solve is bit-identical to the GPU-order oracle, and raises the same
exceptions."""
import numpy as np
import pytest

import oracle_ffi as orc
from paper_1903_10977_b200 import CaseConfig, SmootherConfig, build_case

STAR = dict(geometry="star(0.037, 0.011, 0.5, 0.1, 5)", origin=(-1, -1, 0), extent=(2, 2, 1),
            resolution=(16, 16, 1), family="lagrange", degree=2, levels=2)


def _star(gamma):
    return build_case(CaseConfig(smoother=SmootherConfig("additive-schwarz", gamma=gamma), **STAR))


def test_damped_two_level_richardson_contracts():
    c = _star(0.25)
    st, x, res, it, _ = orc.richardson(c.levels_c(), c.b, tol=1e-10, maxit=200)
    assert st == 0 and 25 <= it <= 60
    A = c.A.to_scipy()
    assert np.linalg.norm(c.b - A @ x) / np.linalg.norm(c.b) <= 2e-10
    for k in range(len(res) - 3, len(res)):
        assert 0.5 < res[k] / res[k - 1] < 0.6


def test_undamped_additive_richardson_diverges():
    c = _star(1.0)
    st, x, res, it, _ = orc.richardson(c.levels_c(), c.b, tol=1e-10, maxit=500)
    assert st == 6  # Diverged
    assert len(res) >= 11 and res[-1] > res[0]
    assert all(res[k] > res[k - 1] for k in range(len(res) - 10, len(res)))


@pytest.mark.gpu
@pytest.mark.parametrize("gamma", [0.25, 1.0])
def test_device_richardson_bitwise(gamma):
    from paper_1903_10977_b200 import Diverged, MgHierarchy, richardson
    c = _star(gamma)
    h = MgHierarchy(c)
    st, xo, ro, it, _ = orc.richardson(c.levels_c(), c.b, tol=1e-10, maxit=500, mode=orc.GPU_ORDER)
    try:
        if st == 0:
            x, rep = richardson(h.A, c.b, h, tol=1e-10, maxit=500)
            assert rep.converged and rep.iterations == it
            assert np.array_equal(np.array(rep.residuals), ro)
            assert np.array_equal(x, xo)
        else:
            with pytest.raises(Diverged) as e:
                richardson(h.A, c.b, h, tol=1e-10, maxit=500)
            assert e.value.report.iterations == it
            assert np.array_equal(np.array(e.value.report.residuals), ro)
    finally:
        h.close()


@pytest.mark.gpu
def test_device_richardson_c1_and_graph_vs_host_loop():
    from paper_1903_10977_b200 import MgHierarchy, _ffi, build_case, configs, richardson
    c = build_case(configs.c1())
    h = MgHierarchy(c)
    try:
        st, xo, ro, it, _ = orc.richardson(c.levels_c(), c.b, tol=1e-8, maxit=300, mode=orc.GPU_ORDER)
        assert st == 0
        x, rep = richardson(h.A, c.b, h, tol=1e-8, maxit=300)
        assert rep.iterations == it and np.array_equal(x, xo)
        _ffi.gpu().ig_set_option(_ffi.IG_OPT_USE_GRAPH, 0)
        try:
            x2, rep2 = richardson(h.A, c.b, h, tol=1e-8, maxit=300)
        finally:
            _ffi.gpu().ig_set_option(_ffi.IG_OPT_USE_GRAPH, 1)
        assert np.array_equal(x, x2) and rep.residuals == rep2.residuals
    finally:
        h.close()
