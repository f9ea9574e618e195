"""Host setup (C++ restatement of the reference's mesh/basis/assembly/
multigrid setup) against the reference's own known answers.  CPU only."""
import ctypes as C

import numpy as np
import pytest
import scipy.sparse as sp

from paper_1903_10977_b200 import CaseConfig, SmootherConfig, _ffi, build_case, configs


def n_dofs(**kw):
    cfg = CaseConfig(**kw).to_c()
    eta, cut, n = C.c_double(), C.c_int64(), C.c_int32()
    assert _ffi.host().igh_eta(C.byref(cfg), C.byref(eta), C.byref(cut), C.byref(n)) == 0
    return n.value, eta.value, cut.value


UNIT = dict(origin=(-1, -1, 0), extent=(2, 2, 1))


@pytest.mark.parametrize("family,p,expected", [("lagrange", 2, 1089), ("bspline", 2, 324),
                                               ("lagrange", 1, 289), ("bspline", 3, 361)])
def test_anchor_counts_untrimmed_16(family, p, expected):
    """proj/tests/test_basis.cpp:79-90."""
    assert n_dofs(geometry="constant(1)", resolution=(16, 16, 1), family=family, degree=p, **UNIT)[0] == expected


def test_trimmed_counts_of_reference_cases():
    """tiny_star n == 111 (proj/tests/test_runner.cpp:120) and star2d n == 347 (:435)."""
    assert n_dofs(geometry="star(0.037, 0.011, 0.5, 0.1, 5)", resolution=(8, 8, 1), family="lagrange",
                  degree=2, **UNIT)[0] == 111
    assert n_dofs(geometry="star(0, 0, 0.5, 0.1, 5)", resolution=(16, 16, 1), family="lagrange", degree=2,
                  **UNIT)[0] == 347


def test_c1_hierarchy_sizes(c1_case):
    """669 / 219 / 87 / 36 DOFs, 15,081 nnz."""
    assert c1_case.level_dofs() == [36, 87, 219, 669]
    assert c1_case.A.nnz == 15081
    assert c1_case.info.coarse_rank <= 36


def test_block_damping_2d_and_3d(c1_case, d3_case):
    """max N_K == 9 for 2D p=2 (proj/tests/test_smoothers.cpp:91); (p+1)^3 = 27 in 3D."""
    for l in range(1, c1_case.n_levels):
        assert c1_case.info.max_nk[l] == 9
        assert c1_case.gamma(l) == 1.0 / 9
    for l in range(1, d3_case.n_levels):
        assert d3_case.info.max_nk[l] == 27
        assert d3_case.gamma(l) == 1.0 / 27


def test_assembled_operator_symmetric_positive_diagonal(c1_case, d3_case):
    for case in (c1_case, d3_case):
        A = case.A.to_scipy()
        assert abs(A - A.T).max() == 0.0
        assert A.diagonal().min() > 0.0
        assert np.all(np.isfinite(A.data)) and np.all(np.isfinite(case.b))


@pytest.mark.parametrize("family", ["bspline", "lagrange"])
def test_restriction_partition_of_unity(family):
    """Coarse basis = R * fine basis; on an untrimmed mesh the coarse partition
    of unity forces every column sum of R to 1 (cf. proj/tests/test_basis.cpp:206-271)."""
    case = build_case(CaseConfig(geometry="constant(1)", resolution=(16, 16, 1), family=family, degree=2,
                                 levels=3, **UNIT))
    for l in (1, 2):
        R = case.level_R(l).to_scipy()
        assert np.max(np.abs(np.asarray(R.sum(axis=0)).ravel() - 1.0)) <= 1e-12


@pytest.mark.parametrize("family", ["bspline", "lagrange"])
def test_galerkin_equals_reassembly_uncut(family):
    """proj/tests/test_multigrid.cpp:85-102: R A R^T equals the coarse assembly
    (with the fine-level penalty) to 1e-11 on an untrimmed mesh."""
    fine = build_case(CaseConfig(geometry="constant(1)", resolution=(16, 16, 1), family=family, degree=2,
                                 levels=3, **UNIT))
    beta = 2.0 / (2.0 / 16)
    for l, res in ((1, 8), (0, 4)):
        direct = build_case(CaseConfig(geometry="constant(1)", resolution=(res, res, 1), family=family, degree=2,
                                       levels=1, beta=beta, **UNIT)).A.to_scipy().toarray()
        gal = fine.level_A(l).to_scipy().toarray()
        assert np.max(np.abs(gal - direct)) <= 1e-11 * np.max(np.abs(direct))


def test_pstrf_matches_lapack():
    """Coarse factor restatement (multigrid.cpp:57-73) vs LAPACK dpstrf (scipy)."""
    from scipy.linalg.lapack import dpstrf
    rng = np.random.default_rng(5)
    for n, r in ((30, 30), (40, 33), (12, 5)):
        B = rng.standard_normal((n, r))
        A = B @ B.T
        tol = 1e-14 * np.max(np.diag(A))
        a = np.asfortranarray(A.copy())
        piv = np.zeros(n, np.int32)
        rank = _ffi.host().igh_pstrf(n, a.ctypes.data_as(C.POINTER(C.c_double)),
                                     piv.ctypes.data_as(C.POINTER(C.c_int32)), tol)
        c, piv_ref, rank_ref, info = dpstrf(A, tol=tol, lower=1)
        assert rank == rank_ref
        assert np.array_equal(piv[:rank], piv_ref[:rank])
        L = np.tril(a)[:rank, :rank]
        assert np.max(np.abs(L - np.tril(c)[:rank, :rank])) <= 1e-10 * np.max(np.abs(L))


def test_coarse_rank_full_on_uncut_and_bounded_on_cut(c1_case):
    """proj/tests/test_multigrid.cpp:55-83."""
    uncut = build_case(CaseConfig(geometry="constant(1)", resolution=(16, 16, 1), family="lagrange", degree=2,
                                  levels=3, **UNIT))
    assert uncut.info.coarse_rank == uncut.level_dofs()[0]
    assert c1_case.info.coarse_rank <= c1_case.level_dofs()[0]


def test_resolution_error():
    from paper_1903_10977_b200 import ResolutionError
    with pytest.raises(ResolutionError):
        build_case(CaseConfig(geometry="constant(1)", resolution=(12, 12, 1), levels=4, **UNIT))


def test_block_factors_invert_the_blocks(c1_case):
    """proj/tests/test_smoothers.cpp:191-213: L L^T reproduces the (filtered) block."""
    A = c1_case.level_A(3).to_scipy().toarray()
    ptr, dofs, fptr, fac = c1_case.blocks(3)
    for b in range(len(ptr) - 1):
        s = ptr[b + 1] - ptr[b]
        d = dofs[ptr[b]:ptr[b + 1]]
        L = np.tril(fac[fptr[b]:fptr[b + 1]].reshape(s, s, order="F"))
        Ab = A[np.ix_(d, d)]
        assert np.max(np.abs(L @ L.T - Ab)) <= 1e-12 * max(np.max(np.abs(Ab)), 1e-300) + 1e-300


def test_blocks_are_owner_ordered_supersets_of_singletons(c1_case):
    """smoothers.cpp:20-67: one block per B-spline DOF, ascending members; every
    DOF covered."""
    for l in range(1, c1_case.n_levels):
        ptr, dofs, _, _ = c1_case.blocks(l)
        n = c1_case.level_dofs()[l]
        assert len(ptr) - 1 == n
        covered = np.zeros(n, bool)
        for b in range(n):
            m = dofs[ptr[b]:ptr[b + 1]]
            assert np.all(np.diff(m) > 0)
            covered[m] = True
        assert covered.all()


def test_igh_file_roundtrip(c1_case, tmp_path):
    path = str(tmp_path / "c1.igh")
    c1_case.write(path)
    from paper_1903_10977_b200 import Case
    back = Case.read(path)
    assert back.level_dofs() == c1_case.level_dofs()
    assert np.array_equal(back.b, c1_case.b)
    for l in range(c1_case.n_levels):
        a, b = c1_case.level_A(l), back.level_A(l)
        assert np.array_equal(a.val, b.val) and np.array_equal(a.col_idx, b.col_idx)
    La, pa, ra = c1_case.coarse()
    Lb, pb, rb = back.coarse()
    assert ra == rb and np.array_equal(pa, pb) and np.array_equal(La, Lb)


def test_seed_offsets_match_survey():
    """SURVEY.md App. B seed-1 values."""
    from paper_1903_10977_b200 import seed_offsets
    assert seed_offsets(1) == [0.0013312315034456172, 0.004915635145254022, 0.009420055071735925]


def test_c3_hole_recipe():
    """64 non-overlapping holes, gap >= 0.01."""
    import re
    geo = configs.c3_geometry(1)
    discs = [tuple(map(float, m)) for m in re.findall(r"disc\(([^,]+), ([^,]+), ([^)]+)\)", geo)]
    assert len(discs) == 64
    for i in range(64):
        for j in range(i):
            (x1, y1, r1), (x2, y2, r2) = discs[i], discs[j]
            assert np.hypot(x1 - x2, y1 - y2) - r1 - r2 >= 0.01


def test_3d_hierarchy_shapes(d3_case):
    assert d3_case.level_dofs()[0] == 216
    for l in range(1, d3_case.n_levels):
        R = d3_case.level_R(l)
        assert R.shape == (d3_case.level_dofs()[l - 1], d3_case.level_dofs()[l])
    assert 0 < d3_case.info.eta < 1


def test_prefilter_layout_matches_post_filter(c1_case):
    """igh_prefilter_blocks (the input of the device factorisation): same block
    count as the post-filter layout, every kept DOF list a subsequence of its
    pre-filter list, and the difference is exactly the filtered-DOF count."""
    for l in range(1, c1_case.n_levels):
        bp, bd = c1_case.prefilter_blocks(l)
        hp, hd, _, _ = c1_case.blocks(l)
        assert bp.shape == hp.shape and bp[0] == 0
        removed = 0
        for b in range(bp.shape[0] - 1):
            pre = list(bd[bp[b]:bp[b + 1]])
            post = list(hd[hp[b]:hp[b + 1]])
            it = iter(pre)
            assert all(d in it for d in post)  # ordered subsequence
            assert pre == sorted(pre)
            removed += len(pre) - len(post)
        assert removed == c1_case.info.filtered_dofs[l]
    with pytest.raises(ValueError):
        c1_case.prefilter_blocks(0)
