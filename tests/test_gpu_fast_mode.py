"""Tolerance mode (SURVEY.md §7.3 "fast mode"): the coarse solve as an
explicit-inverse GEMV (IG_OPT_FAST_COARSE) instead of the oracle-order
substitutions.  Not bit-identical by construction, so it is held to the
north-star tolerances against the sequential-order oracle -- iterations +-1,
residual history 1e-9 over the first 10 iterations, x within 1e-8 in relative
L2, energy norm and non-sliver per-DOF error (tests/parity.py) -- on every
BASELINE config, including C5's rank-deficient coarse matrix.  Strict mode
stays the default and the CI parity bar (bit-identical)."""
import numpy as np
import pytest

import oracle_ffi as orc
from parity import assert_history_close, assert_solution_close

pytestmark = pytest.mark.gpu


def _fast_hierarchy(case):
    from paper_1903_10977_b200 import MgHierarchy, _ffi
    lib = _ffi.gpu()
    assert lib.ig_set_option(_ffi.IG_OPT_FAST_COARSE, 1) == 0
    try:
        return MgHierarchy(case)
    finally:
        lib.ig_set_option(_ffi.IG_OPT_FAST_COARSE, 0)


def _check(case):
    from paper_1903_10977_b200 import pcg
    h = _fast_hierarchy(case)
    try:
        x, rep = pcg(h.A, case.b, h, tol=1e-8, maxit=1000)
        assert rep.converged
        st, xs, rs, its, _ = orc.pcg(case.levels_c(), case.b, tol=1e-8, maxit=1000, mode=orc.SEQ)
        assert st == 0
        assert_history_close(rep.residuals, rs, rep.iterations, its)
        err = assert_solution_close(case, x, xs)
        # the coarse solve alone, against the oracle's substitutions
        lv = case.levels_c()
        r = np.random.default_rng(3).uniform(-1, 1, case.level_dofs()[0])
        xc, xo = h.coarse_solve(r), orc.coarse_solve(lv, r)
        assert np.linalg.norm(xc - xo) <= 1e-8 * np.linalg.norm(xo)
        return rep.iterations, err
    finally:
        h.close()


@pytest.mark.parametrize("name", ["c1_case", "d3_case", "star_case"])
def test_fast_coarse_small(request, name):
    print(name, _check(request.getfixturevalue(name)))


@pytest.mark.parametrize("cfg", ["c2", "c3", "c4", "c5"])
def test_fast_coarse_full_size(cfg):
    from paper_1903_10977_b200 import build_case, configs
    make = {"c2": lambda: configs.c2(p=2, seed=configs.c2_seed()), "c3": configs.c3, "c4": configs.c4,
            "c5": configs.c5}[cfg]
    print(cfg, _check(build_case(make())))
