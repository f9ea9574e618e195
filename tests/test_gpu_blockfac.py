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
