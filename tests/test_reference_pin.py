"""The oracle pinned against THE REFERENCE'S OWN hot-path code.

oracle/_ref/libimmergrid_ref.so is /root/reference/proj/src/{solvers,
multigrid,smoothers}.cpp compiled unmodified, from where they lie, against the
Eigen / LAPACKE stand-in of oracle/ref_shim (the real libraries are absent
from this image; `make -C oracle ref`, oracle/ref_glue.cpp).  The stand-in
evaluates Eigen's kernels in the plain sequential orders the oracle's ORC_SEQ
mode documents, so what these tests pin is the reference's control flow --
pcg / richardson (solvers.cpp:17-120), vcycle_at / coarse_solve
(multigrid.cpp:77-108), Smoother::apply additive and colored multiplicative /
apply_symmetric (smoothers.cpp:169-214), factorize_blocks' filter loop
(smoothers.cpp:131-162) and the coarsest dpstrf call (multigrid.cpp:57-73) --
executed from the reference's sources on the same hierarchy payload: the
oracle (and the host setup restatement) must agree with it BIT FOR BIT.
Eigen's internal kernel orders stay bounded by tests/test_noise_floor.py.

CPU only.  The library is built in this container and travels to the GPU box
with the snapshot; where it is absent the module is skipped."""
import ctypes as C
import dataclasses

import numpy as np
import pytest

import oracle_ffi as orc
import reference_ffi as ref
from conftest import rng_vec
from paper_1903_10977_b200 import CaseConfig, SmootherConfig, build_case, configs

needs_ref = pytest.mark.skipif(not ref.available(), reason="oracle/_ref/libimmergrid_ref.so not built "
                               "(needs /root/reference at build time)")

STAR = dict(geometry="star(0.037, 0.011, 0.5, 0.1, 5)", origin=(-1, -1, 0), extent=(2, 2, 1),
            resolution=(16, 16, 1), family="lagrange", degree=2, levels=2)


def _cases():
    ms = SmootherConfig("multiplicative-schwarz")
    return {
        "c1": lambda: build_case(configs.c1()),
        "c1-ms": lambda: build_case(dataclasses.replace(configs.c1(), smoother=ms)),
        "3d16": lambda: build_case(configs.c4(res=16, levels=3)),
        "3d16-ms": lambda: build_case(dataclasses.replace(configs.c4(res=16, levels=3), smoother=ms)),
        "star": lambda: build_case(CaseConfig(smoother=SmootherConfig("additive-schwarz"), **STAR)),
        "star-ms": lambda: build_case(CaseConfig(smoother=ms, **STAR)),
        "thb": lambda: build_case(configs.c5(base=32, levels=4)),
        "thb-ms": lambda: build_case(dataclasses.replace(configs.c5(base=32, levels=4), smoother=ms)),
        "c2p3": lambda: build_case(dataclasses.replace(configs.c2(p=3, seed=configs.c2_seed()),
                                                       resolution=(64, 64, 1), levels=4)),
    }


_cache = {}


def _get(name):
    if name not in _cache:
        case = _cases()[name]()
        _cache[name] = (case, ref.RefHierarchy(case.levels_c()))
    return _cache[name]


NAMES = list(_cases().keys())


@needs_ref
@pytest.mark.parametrize("name", NAMES)
def test_pcg_is_the_references_pcg(name):
    """solvers.cpp:17-71 with precond = MgHierarchy::apply: status, iteration
    count, every residual and every entry of x."""
    case, h = _get(name)
    lv = case.levels_c()
    st, x, res, it = h.pcg(case.b, tol=configs.TOL, maxit=configs.MAXIT)
    so, xo, ro, ito, _ = orc.pcg(lv, case.b, tol=configs.TOL, maxit=configs.MAXIT, mode=orc.SEQ)
    assert st == 0 and so == 0
    assert it == ito and len(res) == it + 1
    assert np.array_equal(res, ro)
    assert np.array_equal(x, xo)


@needs_ref
@pytest.mark.parametrize("name", ["c1", "3d16", "star-ms", "thb"])
def test_pcg_budget_exhausted_and_trivial_cases(name):
    """NotConverged carries the partial x and maxit+1 residuals
    (solvers.cpp:67-70); b = 0 and tol >= 1 return early (solvers.cpp:26-39)."""
    case, h = _get(name)
    lv = case.levels_c()
    st, x, res, it = h.pcg(case.b, tol=1e-14, maxit=4)
    so, xo, ro, ito, _ = orc.pcg(lv, case.b, tol=1e-14, maxit=4, mode=orc.SEQ)
    assert st == 1 and so == 1 and it == 4 and ito == 4
    assert np.array_equal(res, ro) and len(res) == 5
    assert np.array_equal(x, xo) and np.max(np.abs(x)) > 0
    z = np.zeros_like(case.b)
    st, x, res, it = h.pcg(z, tol=1e-8, maxit=10)
    so, xo, ro, ito, _ = orc.pcg(lv, z, tol=1e-8, maxit=10, mode=orc.SEQ)
    assert (st, it, list(res)) == (so, ito, list(ro)) == (0, 0, [0.0]) and not x.any() and not xo.any()
    st, x, res, it = h.pcg(case.b, tol=1.0, maxit=10)
    so, xo, ro, ito, _ = orc.pcg(lv, case.b, tol=1.0, maxit=10, mode=orc.SEQ)
    assert (st, it, list(res)) == (so, ito, list(ro)) == (0, 0, [1.0]) and not x.any() and not xo.any()


@needs_ref
def test_pcg_breakdown_on_indefinite_operator():
    """test_solvers.cpp:153-173 through the reference's own Breakdown throw."""
    syn = orc.Synthetic(np.diag([1.0, -1.0]))
    h = ref.RefHierarchy(syn.levels_c())
    b = np.array([0.0, 1.0])
    st, x, res, it = h.pcg(b, tol=1e-10, maxit=10)
    so, xo, ro, ito, _ = orc.pcg(syn.levels_c(), b, tol=1e-10, maxit=10, mode=orc.SEQ)
    assert st == 2 and so == 2
    assert np.array_equal(res, ro[:len(res)]) and len(res) >= 1
    h.close()


@needs_ref
def test_identity_cg_one_step():
    """test_solvers.cpp:47-67."""
    n = 40
    syn = orc.Synthetic(np.eye(n))
    h = ref.RefHierarchy(syn.levels_c())
    b = rng_vec(7, n)
    st, x, res, it = h.pcg(b)
    so, xo, ro, ito, _ = orc.pcg(syn.levels_c(), b, mode=orc.SEQ)
    assert (st, it) == (0, 1) == (so, ito)
    assert np.array_equal(res, ro) and np.array_equal(x, xo)
    h.close()


@needs_ref
@pytest.mark.parametrize("name", NAMES)
def test_vcycle_at_every_level(name):
    """multigrid.cpp:90-108 from every level (l = 0 is coarse_solve)."""
    case, h = _get(name)
    lv = case.levels_c()
    for l in range(lv[1]):
        r = rng_vec(11 + l, h.n(l))
        rc, x = h.vcycle_at(l, r)
        assert rc == 0
        assert np.array_equal(x, orc.vcycle_at(lv, l, r)), (name, l)


@needs_ref
@pytest.mark.parametrize("name", ["c1", "3d16-ms"])
def test_vcycle_at_argument_checks(name):
    """multigrid.cpp:91-96: level out of range and residual size mismatch
    throw std::invalid_argument (IG_INVALID_ARGUMENT at the boundary)."""
    case, h = _get(name)
    lv = case.levels_c()
    n = h.n(lv[1] - 1)
    assert h.vcycle_at(lv[1], np.zeros(n))[0] == 3
    assert h.vcycle_at(-1, np.zeros(n))[0] == 3
    assert h.vcycle_at(lv[1] - 1, np.zeros(n + 1))[0] == 3
    x = np.zeros(n)
    r = np.zeros(n)
    dp = C.POINTER(C.c_double)
    assert orc.lib().orc_vcycle_at(lv[0], lv[1], lv[2], lv[1], r.ctypes.data_as(dp), x.ctypes.data_as(dp)) == 3


@needs_ref
@pytest.mark.parametrize("name", NAMES)
def test_smoother_sweeps(name):
    """Smoother::apply Forward / Reverse on every level (additive:
    smoothers.cpp:174-184; colored multiplicative: :186-208) and
    apply_symmetric (:211-214) against the oracle's composition."""
    case, h = _get(name)
    lv = case.levels_c()
    for l in range(1, lv[1]):
        r = rng_vec(23 + l, h.n(l))
        for d in (0, 1):
            assert np.array_equal(h.smoother_apply(l, r, d), orc.smoother_apply(lv, l, r, d)), (name, l, d)
        x1 = orc.smoother_apply(lv, l, r, 0)
        want = x1 + orc.smoother_apply(lv, l, orc.spmv(lv, l, x1, mode=1, y=r), 1)
        assert np.array_equal(h.smoother_apply_symmetric(l, r), want), (name, l)


@needs_ref
@pytest.mark.parametrize("name", ["c1", "3d16", "star", "thb", "c2p3"])
def test_coarse_solve_and_factor(name):
    """coarse_solve (multigrid.cpp:77-88) and the coarsest factorisation as
    MgHierarchy::build states it (multigrid.cpp:57-73) on the payload's
    coarsest operator: L, piv and rank equal the host setup's."""
    case, h = _get(name)
    lv = case.levels_c()
    r = rng_vec(5, h.n(0))
    assert np.array_equal(h.coarse_solve(r), orc.coarse_solve(lv, r))
    rank, L, piv = ref.coarse_factor(lv[0][0].A)
    Lh, pivh, rankh = case.coarse()
    n = h.n(0)
    assert rank == rankh and np.array_equal(piv, pivh)
    Lr = L.reshape(n, n, order="F")
    assert np.array_equal(np.tril(Lr)[:, :rank], np.tril(Lh)[:, :rank])


@needs_ref
@pytest.mark.parametrize("name", ["c1", "3d16", "star", "thb", "c2p3"])
def test_factorize_blocks_filter_loop(name):
    """The reference's factorize_blocks (smoothers.cpp:131-162: gather,
    eigen-filter while lambda_min < ratio * max diag, LLT) on the PRE-filter
    layout gives the host setup's post-filter member lists and factor bits."""
    case, h = _get(name)
    lv = case.levels_c()
    for l in range(1, lv[1]):
        ptr, dofs = case.prefilter_blocks(l)
        st, optr, odofs, fptr, fac = ref.factorize_blocks(lv[0][l].A, ptr, dofs, 1e-16)
        assert st == 0
        hp, hd, hf, hfac = case.blocks(l)
        assert np.array_equal(optr, hp) and np.array_equal(odofs, hd)
        assert np.array_equal(fptr, hf)
        # lower triangles (the upper one is never read)
        for b in range(len(optr) - 1):
            s = optr[b + 1] - optr[b]
            a = fac[fptr[b]:fptr[b + 1]].reshape(s, s, order="F")
            c = hfac[hf[b]:hf[b + 1]].reshape(s, s, order="F")
            assert np.array_equal(np.tril(a), np.tril(c)), (name, l, b)


@needs_ref
def test_factorize_blocks_drops_dofs_and_empties():
    """A filter-active block (a numerically dependent DOF is dropped from that
    block only) and EmptyBlockAfterFilter (smoothers.cpp:146-147)."""
    from paper_1903_10977_b200 import _ffi
    e = 1e-20
    A = np.array([[1.0, 1.0, 0.0], [1.0, 1.0 + e, 0.0], [0.0, 0.0, 2.0]])
    syn = orc.Synthetic(A + np.eye(3) * 0.0)
    Ac = syn.lv[0].A
    ptr = np.array([0, 3], np.int32)
    dofs = np.array([0, 1, 2], np.int32)
    st, optr, odofs, fptr, fac = ref.factorize_blocks(Ac, ptr, dofs, 1e-12)
    assert st == 0 and optr[1] == 2 and 2 in odofs
    # host restatement on the same input
    lib = _ffi.host()
    if hasattr(lib, "igh_factorize_blocks"):
        from paper_1903_10977_b200 import SpMat, factorize_blocks
        hp, hd, hf, hfac = factorize_blocks(SpMat.from_c(Ac, syn), ptr, dofs, 1e-12)
        assert np.array_equal(hp, optr) and np.array_equal(hd, odofs)
        assert np.array_equal(np.tril(hfac.reshape(2, 2, order="F")), np.tril(fac.reshape(2, 2, order="F")))
    neg = orc.Synthetic(np.array([[-1.0]]))
    st, *_ = ref.factorize_blocks(neg.lv[0].A, np.array([0, 1], np.int32), np.array([0], np.int32), 1e-16)
    assert st == 7


def _star(gamma):
    return build_case(CaseConfig(smoother=SmootherConfig("additive-schwarz", gamma=gamma), **STAR))


@needs_ref
@pytest.mark.parametrize("gamma,maxit,want", [(0.25, 200, 0), (1.0, 500, 6), (0.25, 7, 1)])
def test_richardson_is_the_references_richardson(gamma, maxit, want):
    """solvers.cpp:73-120: converged, Diverged after 10 growths, NotConverged."""
    c = _star(gamma)
    h = ref.RefHierarchy(c.levels_c())
    st, x, res, it = h.richardson(c.b, tol=1e-10, maxit=maxit)
    so, xo, ro, ito, _ = orc.richardson(c.levels_c(), c.b, tol=1e-10, maxit=maxit, mode=orc.SEQ)
    assert st == want and so == want and it == ito
    assert np.array_equal(res, ro)
    if want != 6:  # Diverged carries no x (solvers.cpp:108-112)
        assert np.array_equal(x, xo)
    h.close()


@needs_ref
def test_coarse_rank_deficient_hierarchy():
    """C5's family has a rank-deficient coarsest operator: the reference's
    coarse_solve acts on the accepted pivots only (multigrid.cpp:80-86)."""
    case, h = _get("thb")
    _, _, rank = case.coarse()
    assert ref.lib().ref_coarse_rank(h.h) == rank


# ---- full-size golden records written by the reference's own code ---------
# tests/golden/reference_solves.json (tests/golden/make_reference_golden.py):
# these need no reference at run time, so they also run where the library is
# absent.
def _golden():
    import json
    import os
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "reference_solves.json")
    with open(path) as f:
        return json.load(f)


@pytest.mark.parametrize("name", ["c1", "c2", "c5", "c3"])
def test_oracle_reproduces_reference_golden_full_size(name):
    """BASELINE configs at full size: the sequential-order oracle solve equals
    the record the reference's own pcg wrote (iterations, every residual,
    sha256 of x)."""
    import hashlib
    g = _golden()[name]
    cfg = {"c1": configs.c1, "c2": lambda: configs.c2(p=2, seed=configs.c2_seed()), "c3": configs.c3,
           "c5": configs.c5}[name]()
    case = build_case(cfg)
    assert case.level_dofs() == g["level_dofs"]
    assert hashlib.sha256(case.b.tobytes()).hexdigest() == g["b_sha256"]
    assert hashlib.sha256(np.ascontiguousarray(case.A.val).tobytes()).hexdigest() == g["A_val_sha256"]
    orc.set_threads(0)
    st, x, res, it, _ = orc.pcg(case.levels_c(), case.b, tol=configs.TOL, maxit=configs.MAXIT, mode=orc.SEQ)
    assert st == g["status"] == 0 and it == g["iterations"]
    assert [float(v).hex() for v in res] == g["residuals"]
    assert hashlib.sha256(np.ascontiguousarray(x).tobytes()).hexdigest() == g["x_sha256"]
    assert [float(v).hex() for v in x[g["x_sample_idx"]]] == g["x_sample"]


def test_c4_oracle_golden_is_the_references_output():
    """The north-star config at full size (2.0M DOFs, 115 iterations): the
    committed sequential-order oracle golden (tests/golden/c4_oracle.json, what
    the device is held to in tests/test_gpu_parity.py) equals, bit for bit, the
    record the reference's own pcg wrote for the same hierarchy."""
    import json
    import os
    g = _golden()
    if "c4" not in g:
        pytest.skip("C4 reference record not generated")
    with open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "c4_oracle.json")) as f:
        o = json.load(f)
    r, s = g["c4"], o["seq"]
    assert r["level_dofs"] == o["case"]["level_dofs"]
    assert r["b_sha256"] == o["case"]["b_sha256"] and r["A_val_sha256"] == o["case"]["A_val_sha256"]
    assert r["status"] == s["status"] == 0 and r["iterations"] == s["iterations"] == 115
    assert r["residuals"] == s["residuals"]
    assert r["x_sha256"] == s["x_sha256"] and r["x_sample"] == s["x_sample"] and r["x_fsum2"] == s["x_fsum2"]
