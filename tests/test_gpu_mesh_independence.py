"""North star N1: mesh- and cut-independent iteration counts on the C4 family
(the reference pins the pattern on the Lagrange star in
proj/tests/test_multigrid.cpp:193-223 and the paper claims it).

The device solves every member; its count must equal the sequential-order
oracle's within +-1 where the oracle runs, grow by at most 25 % from 16^3 to
128^3 (additive Schwarz: 100 -> 115), and vary by at most 10 % over the
sphere offsets at a fixed resolution.  The full 8-seed x 4-resolution x 2
smoother table is profiles/r02_n1_iterations.md (profiles/n1_iterations.py).
"""
import dataclasses

import pytest

import oracle_ffi as orc

pytestmark = pytest.mark.gpu


def _solve(res, seed, ms=False, oracle=True):
    from paper_1903_10977_b200 import MgHierarchy, SmootherConfig, build_case, configs, pcg
    cfg = configs.c4(res=res, levels=configs.c4_levels(res), seed=seed)
    if ms:
        cfg = dataclasses.replace(cfg, smoother=SmootherConfig("multiplicative-schwarz"))
    case = build_case(cfg)
    h = MgHierarchy(case)
    x, rep = pcg(h.A, case.b, h, tol=1e-8, maxit=1000)
    h.close()
    assert rep.converged
    if oracle:
        st, _, _, it, _ = orc.pcg(case.levels_c(), case.b, tol=1e-8, maxit=1000, mode=orc.SEQ)
        assert st == 0 and abs(it - rep.iterations) <= 1, (res, seed, it, rep.iterations)
    return rep.iterations


def test_additive_mesh_independence():
    its = {res: _solve(res, 1, oracle=res <= 64) for res in (16, 32, 64, 128)}
    assert max(its.values()) <= 1.25 * min(its.values()), its
    assert its[128] == 115  # the C4 golden


def test_additive_cut_independence():
    its = [_solve(32, seed) for seed in (1, 2, 3, 4, 5, 6)]
    assert max(its) <= 1.10 * min(its), its


def test_multiplicative_mesh_and_cut_independence():
    mesh = {res: _solve(res, 1, ms=True, oracle=res <= 32) for res in (16, 32, 64)}
    assert max(mesh.values()) <= 1.25 * min(mesh.values()), mesh
    cut = [_solve(32, seed, ms=True, oracle=False) for seed in (1, 2, 3, 4)]
    assert max(cut) <= 1.10 * min(cut), cut
