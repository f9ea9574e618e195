"""The CPU oracle (checker) against the reference's own solve-path tests
(proj/tests/test_solvers.cpp, test_multigrid.cpp, test_smoothers.cpp) and
against the committed golden fixtures.  CPU only."""
import json
import os

import numpy as np
import pytest

import oracle_ffi as orc
from conftest import rng_vec

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def dense(M):
    return M.to_scipy().toarray()


def test_identity_cg_converges_in_one_step():
    """test_solvers.cpp:47-67."""
    n = 40
    syn = orc.Synthetic(np.eye(n))
    b = rng_vec(7, n)
    st, x, res, it, _ = orc.pcg(syn.levels_c(), b)
    assert st == 0 and it == 1 and len(res) == 2 and res[0] == 1.0 and res[1] <= 1e-14
    assert np.max(np.abs(x - b)) <= 1e-14
    st, x, res, it, _ = orc.pcg(syn.levels_c(), np.zeros(n))
    assert st == 0 and np.max(np.abs(x)) == 0.0 and list(res) == [0.0]


def test_indefinite_operator_breaks_down():
    """test_solvers.cpp:153-173."""
    syn = orc.Synthetic(np.diag([1.0, -1.0]))
    st, x, res, it, _ = orc.pcg(syn.levels_c(), np.array([0.0, 1.0]))
    assert st == 2 and len(res) >= 1


def test_exhausted_budget_reports_partial_state(star_case):
    """test_solvers.cpp:92-107."""
    st, x, res, it, _ = orc.pcg(star_case.levels_c(), star_case.b, tol=1e-10, maxit=5)
    assert st == 1 and it == 5 and len(res) == 6 and np.max(np.abs(x)) > 0


def test_mg_cg_matches_direct_solve(star_case):
    """test_solvers.cpp:69-90: converges, the recomputed residual is <= 2 tol and
    x agrees with a direct solve to 1e-7 (clean star, Lagrange p=2)."""
    tol = 1e-10
    st, x, res, it, _ = orc.pcg(star_case.levels_c(), star_case.b, tol=tol)
    assert st == 0 and it >= 1 and res[0] == 1.0 and len(res) == it + 1
    A = dense(star_case.A)
    b = star_case.b
    assert np.linalg.norm(b - A @ x) / np.linalg.norm(b) <= 2 * tol
    xd = np.linalg.solve(A, b)
    assert np.max(np.abs(x - xd)) <= 1e-7 * np.max(np.abs(xd))


def materialize(f, n):
    M = np.zeros((n, n))
    e = np.zeros(n)
    for j in range(n):
        e[j] = 1.0
        M[:, j] = f(e)
        e[j] = 0.0
    return M


def test_vcycle_is_symmetric_positive_definite(star_case):
    """test_multigrid.cpp:104-115."""
    lv = star_case.levels_c()
    n = star_case.n
    B = materialize(lambda v: orc.vcycle_at(lv, star_case.n_levels - 1, v), n)
    assert np.max(np.abs(B - B.T)) <= 1e-10 * np.max(np.abs(B))
    assert np.linalg.eigvalsh(0.5 * (B + B.T)).min() > 0.0


def test_one_level_hierarchy_is_a_direct_solve():
    """test_multigrid.cpp:172-191."""
    from paper_1903_10977_b200 import CaseConfig, build_case
    case = build_case(CaseConfig(geometry="star(0.037, 0.011, 0.5, 0.1, 5)", origin=(-1, -1, 0),
                                 extent=(2, 2, 1), resolution=(8, 8, 1), family="lagrange", degree=2, levels=1))
    lv = case.levels_c()
    A = dense(case.A)
    r = rng_vec(3, case.n)
    x = orc.vcycle_at(lv, 0, r)
    xd = np.linalg.solve(A, r)
    assert np.max(np.abs(x - xd)) <= 1e-9 * np.max(np.abs(xd))
    assert np.max(np.abs(orc.vcycle_at(lv, 0, np.zeros(case.n)))) == 0.0


def test_additive_schwarz_equals_explicit_block_loop(c1_case):
    """test_smoothers.cpp:261-291."""
    from scipy.linalg import cho_solve
    lv = c1_case.levels_c()
    for l in range(1, c1_case.n_levels):
        ptr, dofs, fptr, fac = c1_case.blocks(l)
        r = rng_vec(9 + l, c1_case.level_dofs()[l])
        x = np.zeros_like(r)
        for b in range(len(ptr) - 1):
            s = ptr[b + 1] - ptr[b]
            d = dofs[ptr[b]:ptr[b + 1]]
            L = np.tril(fac[fptr[b]:fptr[b + 1]].reshape(s, s, order="F"))
            x[d] += cho_solve((L, True), r[d])
        x *= c1_case.gamma(l)
        xo = orc.as_apply(lv, l, r)
        assert np.linalg.norm(xo - x) <= 1e-12 * np.linalg.norm(x)


def test_damped_additive_schwarz_is_a_contraction():
    """test_smoothers.cpp:347-367: lambda_max(gamma M^-1 A) <= 1 + 1e-10."""
    from paper_1903_10977_b200 import CaseConfig, SmootherConfig, build_case
    case = build_case(CaseConfig(geometry="star(0.037, 0.011, 0.5, 0.1, 5)", origin=(-1, -1, 0),
                                 extent=(2, 2, 1), resolution=(8, 8, 1), family="bspline", degree=2, levels=2,
                                 smoother=SmootherConfig("additive-schwarz")))
    lv = case.levels_c()
    A = dense(case.A)
    MA = materialize(lambda v: orc.as_apply(lv, 1, A @ v), case.n)
    assert np.max(np.real(np.linalg.eigvals(MA))) <= 1 + 1e-10


def test_two_level_error_propagation_factorises_uncut():
    """test_multigrid.cpp:117-170 (uncut: 1e-11):
    I - B A = (I - M A)(I - R^T A_c^-1 R A)(I - M A)."""
    from paper_1903_10977_b200 import CaseConfig, build_case
    case = build_case(CaseConfig(geometry="constant(1)", origin=(-1, -1, 0), extent=(2, 2, 1),
                                 resolution=(8, 8, 1), family="lagrange", degree=2, levels=2))
    lv = case.levels_c()
    n = case.n
    A = dense(case.A)
    R = dense(case.level_R(1))
    Ac = dense(case.level_A(0))
    I = np.eye(n)
    E = I - materialize(lambda v: orc.vcycle_at(lv, 1, A @ v), n)
    MA = materialize(lambda v: orc.as_apply(lv, 1, A @ v), n)
    C = I - R.T @ np.linalg.solve(Ac, R @ A)
    ref = (I - MA) @ C @ (I - MA)
    assert np.max(np.abs(E - ref)) <= 1e-11 * max(1.0, np.max(np.abs(ref)))


def test_reduction_orders_agree_within_north_star_tolerance(c1_case):
    lv = c1_case.levels_c()
    s0, x0, r0, i0, _ = orc.pcg(lv, c1_case.b, tol=1e-8, mode=orc.SEQ)
    s1, x1, r1, i1, _ = orc.pcg(lv, c1_case.b, tol=1e-8, mode=orc.GPU_ORDER)
    assert s0 == s1 == 0 and abs(i0 - i1) <= 1
    k = min(11, len(r0), len(r1))
    assert np.all(np.abs(r0[:k] - r1[:k]) <= 1e-9 * r0[:k])
    assert np.linalg.norm(x0 - x1) <= 1e-8 * np.linalg.norm(x0)


def test_gpu_order_dot_is_the_documented_tree():
    """orc_dot(GPU_ORDER) == chunked tree of oracle.h, restated in numpy."""
    a = rng_vec(1, 70001)
    b = rng_vec(2, 70001)
    prod = a * b

    def tree256(v):
        w = []
        for g in range(8):
            lane = v[32 * g:32 * g + 32].copy()
            for off in (16, 8, 4, 2, 1):
                lane = lane + lane[np.arange(32) ^ off]
            w.append(lane[0])
        return ((w[0] + w[1]) + (w[2] + w[3])) + ((w[4] + w[5]) + (w[6] + w[7]))

    nc = (len(prod) + 255) // 256
    pad = np.zeros(nc * 256)
    pad[:len(prod)] = prod
    P = np.array([tree256(pad[256 * c:256 * c + 256]) for c in range(nc)])
    acc = np.zeros(256)
    for t in range(256):
        s = 0.0
        for k in range(t, nc, 256):
            s = s + P[k]
        acc[t] = s
    assert orc.dot(orc.GPU_ORDER, a, b) == tree256(acc)


def _hex(a):
    return np.array([float.fromhex(h) for h in a])


def test_oracle_reproduces_c1_golden(c1_case):
    """Regression pin: host setup + oracle reproduce tests/golden/c1_oracle.json bit for bit."""
    with open(os.path.join(GOLDEN, "c1_oracle.json")) as f:
        g = json.load(f)
    assert c1_case.level_dofs() == g["case"]["level_dofs"]
    import hashlib
    assert hashlib.sha256(c1_case.b.tobytes()).hexdigest() == g["case"]["b_sha256"]
    assert hashlib.sha256(np.ascontiguousarray(c1_case.A.val).tobytes()).hexdigest() == g["case"]["A_val_sha256"]
    for key, mode in (("gpu_order", orc.GPU_ORDER), ("seq", orc.SEQ)):
        st, x, res, it, _ = orc.pcg(c1_case.levels_c(), c1_case.b, tol=1e-8, mode=mode)
        assert st == g[key]["status"] and it == g[key]["iterations"]
        assert np.array_equal(res, _hex(g[key]["residuals"]))
        assert np.array_equal(x, _hex(g[key]["x"]))


@pytest.mark.slow
def test_c4_host_setup_matches_golden_signature():
    """Full-size C4 (configs[3]) host setup reproduces the hierarchy the
    committed C4 golden solve was computed on (sizes, rhs and operator checksums)."""
    path = os.path.join(GOLDEN, "c4_oracle.json")
    if not os.path.exists(path):
        pytest.skip("c4 golden not generated")
    from paper_1903_10977_b200 import build_case, configs
    with open(path) as f:
        g = json.load(f)
    case = build_case(configs.c4())
    assert case.level_dofs() == g["case"]["level_dofs"]
    assert [int(case.info.nnz[k]) for k in range(case.n_levels)] == g["case"]["nnz"]
    import hashlib
    assert hashlib.sha256(case.b.tobytes()).hexdigest() == g["case"]["b_sha256"]
    assert hashlib.sha256(np.ascontiguousarray(case.A.val).tobytes()).hexdigest() == g["case"]["A_val_sha256"]
    assert g["gpu_order"]["status"] == 0 and g["seq"]["status"] == 0
    assert abs(g["gpu_order"]["iterations"] - g["seq"]["iterations"]) <= 1
