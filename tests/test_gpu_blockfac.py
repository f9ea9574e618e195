"""Device batched Schwarz block factorisation (
csrc/blockfac.cuh): eigen-filter + LLT of every pre-filter block on the GPU
must reproduce the host hierarchy's post-filter layout BIT FOR BIT (kept DOFs,
pointers, factor value bits) -- make_smoother's factorize_blocks,
proj/src/smoothers.cpp:131-162."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _check(case, ratio):
    from paper_1903_10977_b200 import factorize_blocks
    tot_filtered = 0
    for l in range(1, case.n_levels):
        bp, bd = case.prefilter_blocks(l)
        optr, odofs, ofp, ofac, filt, (wall, dev) = factorize_blocks(case.level_A(l), bp, bd, ratio)
        hptr, hdofs, hfp, hfac = case.blocks(l)
        assert np.array_equal(optr, hptr), f"level {l}: block pointers"
        assert np.array_equal(odofs, hdofs), f"level {l}: kept DOFs"
        assert np.array_equal(ofp, hfp), f"level {l}: factor pointers"
        assert np.array_equal(ofac.view(np.uint64), np.asarray(hfac).view(np.uint64)), f"level {l}: factor bits"
        assert filt == case.info.filtered_dofs[l]
        tot_filtered += filt
    return tot_filtered


@pytest.mark.parametrize("case_name", ["c1_case", "d3_case", "star_case"])
def test_blockfac_bitwise(request, case_name):
    _check(request.getfixturevalue(case_name), 1e-16)


def test_blockfac_filter_active():
    """A filter ratio that removes DOFs (the eigen-filter loop with Jacobi
    sweeps and repeated re-gathers runs on many blocks)."""
    from paper_1903_10977_b200 import CaseConfig, SmootherConfig, build_case, configs
    cfg = configs.c1()
    cfg = CaseConfig(**{**cfg.__dict__, "smoother": SmootherConfig("additive-schwarz", filter_ratio=1e-3)})
    case = build_case(cfg)
    assert _check(case, 1e-3) > 0


def test_blockfac_thb_full_size():
    from paper_1903_10977_b200 import build_case, configs
    _check(build_case(configs.c5()), 1e-16)


def test_blockfac_c4_full_size():
    from paper_1903_10977_b200 import build_case, configs
    case = build_case(configs.c4())
    from paper_1903_10977_b200 import factorize_blocks
    l = case.n_levels - 1
    bp, bd = case.prefilter_blocks(l)
    optr, odofs, ofp, ofac, filt, (wall, dev) = factorize_blocks(case.level_A(l), bp, bd, 1e-16)
    hptr, hdofs, hfp, hfac = case.blocks(l)
    assert np.array_equal(optr, hptr) and np.array_equal(odofs, hdofs) and np.array_equal(ofp, hfp)
    assert np.array_equal(ofac.view(np.uint64), np.asarray(hfac).view(np.uint64))
    print(f"C4 finest block factorisation: {len(bp) - 1} blocks, device {dev * 1e3:.1f} ms, wall {wall:.2f} s")


def test_blockfac_all_filtered_is_an_error(c1_case):
    """A block that loses every DOF raises (the reference's runtime_error)."""
    from paper_1903_10977_b200 import factorize_blocks
    A = c1_case.level_A(c1_case.n_levels - 1)
    with pytest.raises(ValueError):
        factorize_blocks(A, np.array([0, 2], np.int32), np.array([0, 1], np.int32), 1e300)


def _pstrf_both(A, tol):
    import ctypes as C
    from paper_1903_10977_b200 import _ffi
    n = A.shape[0]
    ah = np.asfortranarray(A.copy())
    ad = np.asfortranarray(A.copy())
    ph = np.zeros(max(n, 1), np.int32)
    pd = np.zeros(max(n, 1), np.int32)
    dp, ip = C.POINTER(C.c_double), C.POINTER(C.c_int32)
    rh = _ffi.host().igh_pstrf(n, ah.ctypes.data_as(dp), ph.ctypes.data_as(ip), tol)
    rd = C.c_int32(-7)
    assert _ffi.gpu().ig_pstrf(n, ad.ctypes.data_as(dp), pd.ctypes.data_as(ip), tol, C.byref(rd)) == 0
    return (rh, ah, ph), (rd.value, ad, pd)


@pytest.mark.parametrize("n,r", [(1, 1), (30, 30), (216, 216), (40, 33), (12, 5), (300, 120)])
def test_device_pstrf_bitwise(n, r):
    """Device dpstf2 (k_pstrf) vs the host restatement igh_pstrf: rank, pivots
    and every entry of the factored array (including the untouched trailing
    part of a rank-deficient factorisation) bit for bit."""
    rng = np.random.default_rng(n * 1000 + r)
    B = rng.standard_normal((n, r))
    A = B @ B.T
    (rh, ah, ph), (rd, ad, pd) = _pstrf_both(A, 1e-14 * np.max(np.diag(A)))
    assert rh == rd
    assert np.array_equal(ph, pd)
    assert np.array_equal(ah.view(np.uint64), ad.view(np.uint64))


def test_device_pstrf_edge_cases():
    for A, tol in ((np.zeros((0, 0)), 0.0), (-np.eye(3), 0.0), (np.full((2, 2), np.nan), 0.0),
                   (np.diag([4.0, 0.0, 1.0]), -1.0)):
        (rh, ah, ph), (rd, ad, pd) = _pstrf_both(A, tol)
        assert rh == rd and np.array_equal(ph, pd)
        assert np.array_equal(ah.view(np.uint64), ad.view(np.uint64))


@pytest.mark.parametrize("case_name", ["c1_case", "d3_case"])
def test_device_pstrf_coarse_levels(request, case_name):
    """The hierarchies' own coarsest operators (sliver cuts: rank-deficient)."""
    case = request.getfixturevalue(case_name)
    A0 = case.level_A(0).to_scipy().toarray()
    (rh, ah, ph), (rd, ad, pd) = _pstrf_both(A0, 1e-14 * np.max(np.diag(A0)))
    assert rh == rd == case.info.coarse_rank
    assert np.array_equal(ph, pd) and np.array_equal(ah.view(np.uint64), ad.view(np.uint64))


def _same_solve(case):
    import oracle_ffi as orc
    from paper_1903_10977_b200 import MgHierarchy, pcg
    hd = MgHierarchy.build_on_device(case)
    try:
        x, rep = pcg(hd.A, case.b, hd, tol=1e-8, maxit=1000)
        st, xo, ro, it, _ = orc.pcg(case.levels_c(), case.b, tol=1e-8, maxit=1000, mode=orc.GPU_ORDER)
        assert st == 0 and rep.iterations == it
        assert np.array_equal(np.array(rep.residuals), ro) and np.array_equal(x, xo)
        for l in range(hd.levels()):
            from conftest import rng_vec
            r = rng_vec(3 + l, hd._n[l])
            assert np.array_equal(hd.vcycle_at(l, r), orc.vcycle_at(case.levels_c(), l, r))
        return hd.setup_seconds
    finally:
        hd.close()


@pytest.mark.parametrize("case_name", ["c1_case", "d3_case", "star_case"])
def test_device_hierarchy_build_solves_identically(request, case_name):
    """ig_hier_build (Galerkin + block factorisation + pstrf on the device,
    then the layouts) gives the host-built hierarchy's V-cycles and PCG solve
    bit for bit (the oracle runs on the host-built payload)."""
    _same_solve(request.getfixturevalue(case_name))


def test_device_hierarchy_build_multiplicative():
    from paper_1903_10977_b200 import CaseConfig, SmootherConfig, build_case, configs
    cfg = configs.c1()
    case = build_case(CaseConfig(**{**cfg.__dict__, "smoother": SmootherConfig("multiplicative-schwarz")}))
    _same_solve(case)


def test_device_hierarchy_build_c4_full_size():
    """Full-size C4: the device-built handle solves exactly like the handle
    built from the host payload (both on the GPU; the C4 oracle solve is
    covered by test_gpu_parity)."""
    from paper_1903_10977_b200 import MgHierarchy, build_case, configs, pcg
    case = build_case(configs.c4())
    hd = MgHierarchy.build_on_device(case)
    wall, dev, create = hd.setup_seconds
    xd, rd = pcg(hd.A, case.b, hd, tol=1e-8, maxit=1000)
    hd.close()
    hh = MgHierarchy(case)
    xh, rh = pcg(hh.A, case.b, hh, tol=1e-8, maxit=1000)
    hh.close()
    assert rd.iterations == rh.iterations == 115
    assert np.array_equal(np.array(rd.residuals), np.array(rh.residuals)) and np.array_equal(xd, xh)
    print(f"C4 device hierarchy build: wall {wall:.2f} s (device kernels {dev * 1e3:.0f} ms, "
          f"ig_hier_create {create:.2f} s); host mg setup {case.info.seconds_mg_setup:.2f} s")
