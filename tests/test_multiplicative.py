"""Multiplicative (colored) Schwarz — SURVEY.md §8(f) row 1, the reference's
default smoother (smoothers.hpp:17).  CPU: host colouring against the
reference's structural bounds and the oracle sweep against the reference's
own algebraic definition (proj/tests/test_smoothers.cpp:153-190, :293-345,
:369-381)."""
import numpy as np
import pytest

import oracle_ffi as orc
from conftest import rng_vec
from paper_1903_10977_b200 import CaseConfig, SmootherConfig, build_case

UNIT = dict(origin=(-1, -1, 0), extent=(2, 2, 1))
MS = SmootherConfig("multiplicative-schwarz")
STAR = "star(0.037, 0.011, 0.5, 0.1, 5)"


def _case(geometry="constant(1)", family="bspline", n=8, levels=2, **kw):
    return build_case(CaseConfig(geometry=geometry, resolution=(n, n, 1), family=family, degree=2, levels=levels,
                                 smoother=MS, **UNIT, **kw))


@pytest.mark.parametrize("family,n,bound,kw", [("lagrange", 8, 4, {}), ("bspline", 8, 9, {}),
                                               ("thb", 16, 18, {"refine_boxes": [(-0.24, -0.24, 0.24, 0.24)]})])
def test_color_bounds_and_disjoint_blocks(family, n, bound, kw):
    """test_smoothers.cpp:153-190: colour count within the structural bound;
    same-colour blocks never share a DOF (they do not even share an element)."""
    c = _case(family=family, n=n, **kw)
    col, nc = c.colors(1)
    assert 1 <= nc <= bound
    ptr, dofs, _, _ = c.blocks(1)
    for k in range(nc):
        members = np.concatenate([dofs[ptr[b]:ptr[b + 1]] for b in np.flatnonzero(col == k)])
        assert len(members) == len(np.unique(members))
    assert c.gamma(1) == 1.0  # undamped by default (smoothers.cpp:234-239)


def _reference_sweep(c, l, r, direction):
    """The test's reference definition (test_smoothers.cpp:293-316): colours in
    sweep order, each block's solve applied to the frozen residual, res -= A dx."""
    A = c.level_A(l).to_scipy()
    ptr, dofs, fptr, fac = c.blocks(l)
    col, nc = c.colors(l)
    x = np.zeros_like(r)
    res = r.copy()
    order = range(nc - 1, -1, -1) if direction == 0 else range(nc)
    for k in order:
        dx = np.zeros_like(r)
        for b in np.flatnonzero(col == k):
            d = dofs[ptr[b]:ptr[b + 1]]
            s = len(d)
            L = np.tril(fac[fptr[b]:fptr[b + 1]].reshape(s, s, order="F"))
            dx[d] = np.linalg.solve(L.T, np.linalg.solve(L, res[d]))
        x += dx
        res -= A @ dx
    return c.gamma(l) * x


@pytest.mark.parametrize("direction", [0, 1])
def test_oracle_sweep_matches_reference_definition(direction):
    c = _case(STAR, family="lagrange", n=16)
    r = rng_vec(11, c.level_dofs()[1])
    xo = orc.smoother_apply(c.levels_c(), 1, r, direction)
    xr = _reference_sweep(c, 1, r, direction)
    assert np.abs(xo - xr).max() <= 1e-12 * np.abs(xr).max()


def test_reverse_is_adjoint_of_forward():
    """test_smoothers.cpp:320-345."""
    c = _case(STAR, family="lagrange", n=16)
    n = c.level_dofs()[1]
    u, v = rng_vec(3, n), rng_vec(4, n)
    lhs = orc.smoother_apply(c.levels_c(), 1, u, 0) @ v
    rhs = u @ orc.smoother_apply(c.levels_c(), 1, v, 1)
    assert abs(lhs - rhs) <= 1e-10 * abs(rhs)


def test_symmetric_double_iteration_is_positive_contraction():
    """test_smoothers.cpp:369-381: (M^-1 + M^-T - M^-T A M^-1) A has spectrum in (0, 1]."""
    c = _case(STAR, family="lagrange", n=8)
    lv = c.levels_c()
    A = c.level_A(1).to_scipy().toarray()
    n = A.shape[0]

    def sym(r):
        x1 = orc.smoother_apply(lv, 1, r, 0)
        return x1 + orc.smoother_apply(lv, 1, r - A @ x1, 1)

    E = np.column_stack([sym(A[:, j]) for j in range(n)])
    w = np.linalg.eigvals(E).real
    assert w.max() <= 1.0 + 1e-10 and w.min() > 0.0


def test_ms_pcg_converges_faster_than_additive():
    geo = dict(geometry="disc(0.5, 0.5, 0.4)", resolution=(32, 32, 1), degree=2, levels=4, origin=(0, 0, 0),
               extent=(1, 1, 1))
    ms = build_case(CaseConfig(smoother=MS, **geo))
    add = build_case(CaseConfig(smoother=SmootherConfig("additive-schwarz"), **geo))
    st1, x1, _, it1, _ = orc.pcg(ms.levels_c(), ms.b, tol=1e-8, maxit=200)
    st2, x2, _, it2, _ = orc.pcg(add.levels_c(), add.b, tol=1e-8, maxit=200)
    assert st1 == 0 and st2 == 0 and it1 < it2
    A = ms.A.to_scipy()
    assert np.linalg.norm(ms.b - A @ x1) <= 2e-8 * np.linalg.norm(ms.b)
