"""Every device SpMV layout gives the SAME bits: the pattern SELL
(spmv_psell.cuh), the row-dictionary SELL thread-per-row kernel and the
group-per-row kernel (kernels.cuh) are selected by size thresholds, so the
small parity cases would only ever see one of them.  Here the thresholds are
forced so each layout runs on every level, and every level product and the
whole PCG solve are compared bit-for-bit with the GPU-order oracle."""
import numpy as np
import pytest

import oracle_ffi as orc
from conftest import rng_vec

pytestmark = pytest.mark.gpu

# (IG_OPT_SMALL_ROWS, IG_OPT_PSELL)
LAYOUTS = {"pattern-sell": (0, 1), "dict-sell": (0, 0), "group-per-row": (1 << 30, 0)}


@pytest.fixture(params=list(LAYOUTS))
def layout(request):
    from paper_1903_10977_b200 import _ffi
    lib = _ffi.gpu()
    small, psell = LAYOUTS[request.param]
    lib.ig_set_option(_ffi.IG_OPT_SMALL_ROWS, small)
    lib.ig_set_option(_ffi.IG_OPT_PSELL, psell)
    lib.ig_set_option(_ffi.IG_OPT_PSELL_PAIRS_ROWS, 0)  # pair / two-line / multi-piece slices on the small cases too
    yield request.param
    lib.ig_set_option(_ffi.IG_OPT_SMALL_ROWS, 12000)
    lib.ig_set_option(_ffi.IG_OPT_PSELL, 1)
    lib.ig_set_option(_ffi.IG_OPT_PSELL_PAIRS_ROWS, 100000)


@pytest.fixture(scope="module")
def c3_small_case():
    """A C3-like perforated plate (Dirichlet on the box edges) at 128^2, 6
    levels: restriction/prolongation shapes whose scaled offset bases exceed
    the column range (regression for the padded-gather bound)."""
    from paper_1903_10977_b200 import CaseConfig, SmootherConfig, build_case, configs
    return build_case(CaseConfig(geometry=configs.c3_geometry(1, holes=8), resolution=(128, 128, 1), degree=2, levels=6,
                                 dirichlet_box_sides=True, smoother=SmootherConfig("additive-schwarz")))


@pytest.mark.parametrize("case_name", ["c1_case", "d3_case", "star_case", "c3_small_case"])
def test_layout_bitwise(request, layout, case_name):
    from paper_1903_10977_b200 import MgHierarchy, pcg
    case = request.getfixturevalue(case_name)
    h = MgHierarchy(case)
    lv = case.levels_c()
    try:
        for l in range(1, h.levels()):
            A, R = h.level(l)
            x = rng_vec(70 + l, A.cols())
            y0 = rng_vec(80 + l, A.rows())
            assert np.array_equal(h.spmv(l, x, 0), orc.spmv(lv, l, x, 0))
            assert np.array_equal(h.spmv(l, x, 1, y0), orc.spmv(lv, l, x, 1, y0))
            assert np.array_equal(h.spmv(l, x, 2), orc.spmv(lv, l, x, 2))
            xc = rng_vec(90 + l, R.rows())
            assert np.array_equal(h.spmv(l, xc, 3), orc.spmv(lv, l, xc, 3))
        x, rep = pcg(h.A, case.b, h, tol=1e-8, maxit=1000)
        st, xo, ro, it, _ = orc.pcg(lv, case.b, tol=1e-8, maxit=1000, mode=orc.GPU_ORDER)
        assert st == 0 and rep.iterations == it
        assert np.array_equal(np.array(rep.residuals), ro)
        assert np.array_equal(x, xo)
    finally:
        h.close()


def test_pattern_sell_nonfinite_and_signed_zero(star_case):
    """Edge values through the pattern layout: -0.0 inputs, a NaN entry and an
    Inf entry of x propagate exactly as in the oracle's row sums."""
    from paper_1903_10977_b200 import MgHierarchy, _ffi
    lib = _ffi.gpu()
    lib.ig_set_option(_ffi.IG_OPT_SMALL_ROWS, 0)
    lib.ig_set_option(_ffi.IG_OPT_PSELL_PAIRS_ROWS, 0)
    try:
        h = MgHierarchy(star_case)
    finally:
        lib.ig_set_option(_ffi.IG_OPT_SMALL_ROWS, 12000)
        lib.ig_set_option(_ffi.IG_OPT_PSELL_PAIRS_ROWS, 100000)
    lv = star_case.levels_c()
    try:
        l = h.levels() - 1
        A, _ = h.level(l)
        x = -np.zeros(A.cols())
        assert np.array_equal(np.signbit(h.spmv(l, x, 0)), np.signbit(orc.spmv(lv, l, x, 0)))
        x = rng_vec(5, A.cols())
        x[3] = np.nan
        x[A.cols() // 2] = np.inf
        yg, yo = h.spmv(l, x, 0), orc.spmv(lv, l, x, 0)
        assert np.array_equal(np.isnan(yg), np.isnan(yo))
        m = ~np.isnan(yo)
        assert np.array_equal(yg[m], yo[m])
    finally:
        h.close()


def test_breakdown_through_pattern_sell():
    """proj/tests/test_solvers.cpp:153-173 with the finest A in the pattern
    layout: p.Ap <= 0 is detected by k_pap (the separate canonical reduction)
    and reported as Breakdown."""
    from paper_1903_10977_b200 import Breakdown, MgHierarchy, _ffi, pcg
    lib = _ffi.gpu()
    lib.ig_set_option(_ffi.IG_OPT_SMALL_ROWS, 0)
    lib.ig_set_option(_ffi.IG_OPT_PSELL_PAIRS_ROWS, 0)
    try:
        h = MgHierarchy(orc.Synthetic(np.diag([1.0, -1.0])))
    finally:
        lib.ig_set_option(_ffi.IG_OPT_SMALL_ROWS, 12000)
        lib.ig_set_option(_ffi.IG_OPT_PSELL_PAIRS_ROWS, 100000)
    try:
        with pytest.raises(Breakdown) as e:
            pcg(h.A, np.array([0.0, 1.0]), h)
        assert len(e.value.report.residuals) >= 1
    finally:
        h.close()


@pytest.mark.parametrize("ab,ctab", [(0, 1), (1, 1), (1, 0)])
@pytest.mark.parametrize("case_name", ["d3_48_case", "c3_small_case", "c1_case"])
def test_pair_item_prolongation_bitwise(request, case_name, ab, ctab):
    """FASTAB slices (IG_OPT_PSELL_AB: a prolongation's row pairs sharing one
    column list, two interleaved value sequences, values from HBM or the
    constant-bank table) against the GENERAL-slice layout: restriction,
    prolongation (+ correction), V-cycles and the solve give the oracle's
    bits (pattern layout forced on every level)."""
    from paper_1903_10977_b200 import MgHierarchy, _ffi, pcg
    lib = _ffi.gpu()
    case = request.getfixturevalue(case_name)
    lv = case.levels_c()
    lib.ig_set_option(_ffi.IG_OPT_PSELL_AB, ab)
    lib.ig_set_option(_ffi.IG_OPT_PSELL_CTAB, ctab)
    lib.ig_set_option(_ffi.IG_OPT_SMALL_ROWS, 0)
    lib.ig_set_option(_ffi.IG_OPT_PSELL_PAIRS_ROWS, 0)
    try:
        h = MgHierarchy(case)
    finally:
        lib.ig_set_option(_ffi.IG_OPT_PSELL_AB, 1)
        lib.ig_set_option(_ffi.IG_OPT_PSELL_CTAB, 1)
        lib.ig_set_option(_ffi.IG_OPT_SMALL_ROWS, 12000)
        lib.ig_set_option(_ffi.IG_OPT_PSELL_PAIRS_ROWS, 100000)
    try:
        for l in range(1, h.levels()):
            A, R = h.level(l)
            x = rng_vec(470 + l, A.cols())
            assert np.array_equal(h.spmv(l, x, 2), orc.spmv(lv, l, x, 2))
            xc = rng_vec(490 + l, R.rows())
            assert np.array_equal(h.spmv(l, xc, 3), orc.spmv(lv, l, xc, 3))
        x, rep = pcg(h.A, case.b, h, tol=1e-8, maxit=1000)
        st, xo, ro, it, _ = orc.pcg(lv, case.b, tol=1e-8, maxit=1000, mode=orc.GPU_ORDER)
        assert st == 0 and rep.iterations == it and np.array_equal(x, xo)
    finally:
        h.close()


@pytest.mark.parametrize("ctab", [0, 1])
def test_constant_value_table_bitwise(ctab):
    """FAST2 value sequences read from the constant-bank kernel-parameter table
    (IG_OPT_PSELL_CTAB) or from HBM give the same bits -- on a THB hierarchy,
    whose prolongation operators also carry FAST2 slices (pattern layout
    forced on every level)."""
    from paper_1903_10977_b200 import MgHierarchy, _ffi, build_case, configs, pcg
    lib = _ffi.gpu()
    case = build_case(configs.c5(base=64, levels=4))
    lib.ig_set_option(_ffi.IG_OPT_PSELL_CTAB, ctab)
    lib.ig_set_option(_ffi.IG_OPT_SMALL_ROWS, 0)
    lib.ig_set_option(_ffi.IG_OPT_PSELL_PAIRS_ROWS, 0)
    try:
        h = MgHierarchy(case)
    finally:
        lib.ig_set_option(_ffi.IG_OPT_PSELL_CTAB, 1)
        lib.ig_set_option(_ffi.IG_OPT_SMALL_ROWS, 12000)
        lib.ig_set_option(_ffi.IG_OPT_PSELL_PAIRS_ROWS, 100000)
    lv = case.levels_c()
    try:
        for l in range(1, h.levels()):
            A, R = h.level(l)
            x = rng_vec(170 + l, A.cols())
            assert np.array_equal(h.spmv(l, x, 0), orc.spmv(lv, l, x, 0))
            xc = rng_vec(190 + l, R.rows())
            assert np.array_equal(h.spmv(l, xc, 3), orc.spmv(lv, l, xc, 3))
        x, rep = pcg(h.A, case.b, h, tol=1e-8, maxit=1000)
        st, xo, ro, it, _ = orc.pcg(lv, case.b, tol=1e-8, maxit=1000, mode=orc.GPU_ORDER)
        assert st == 0 and rep.iterations == it and np.array_equal(x, xo)
    finally:
        h.close()


@pytest.fixture(scope="module")
def d3_48_case():
    """3D C4-like case at 48^3 (x-line runs of ~44 rows: long enough to pair)."""
    from paper_1903_10977_b200 import build_case, configs
    return build_case(configs.c4(res=48, levels=4))


@pytest.mark.parametrize("lines2,multi,rows4,edge", [(0, 0, 1, 0), (1, 0, 0, 1), (0, 1, 1, 1), (1, 1, 0, 0), (1, 1, 1, 1),
                                                     (1, 1, 1, 0)])
def test_two_line_slices_bitwise(d3_48_case, lines2, multi, rows4, edge):
    """FAST4 slices (two x-lines per slice sharing their column runs,
    IG_OPT_PSELL_LINES2) and FAST2M slices (row pairs of up to four short runs
    per slice, per-lane column offsets and load parity, IG_OPT_PSELL_MULTI),
    pattern layout forced on every level: the oracle's bits for the level
    products and the PCG solve under every combination; rows4: the two-line
    slices with four rows of each line per lane (FAST8, IG_OPT_PSELL_ROWS4);
    edge: the x-line end rows as FASTE slices over the edge-compacted copy of
    x (IG_OPT_PSELL_EDGE_ROWS, k_xgather before every product)."""
    from paper_1903_10977_b200 import MgHierarchy, _ffi, pcg
    lib = _ffi.gpu()
    d3_case = d3_48_case
    lv = d3_case.levels_c()
    lib.ig_set_option(_ffi.IG_OPT_PSELL_LINES2, lines2)
    lib.ig_set_option(_ffi.IG_OPT_PSELL_MULTI, multi)
    lib.ig_set_option(_ffi.IG_OPT_PSELL_ROWS4, rows4)
    lib.ig_set_option(_ffi.IG_OPT_PSELL_ROWS4_ROWS, 0)
    lib.ig_set_option(_ffi.IG_OPT_PSELL_EDGE_ROWS, 1 if edge else 0)
    lib.ig_set_option(_ffi.IG_OPT_SMALL_ROWS, 0)
    lib.ig_set_option(_ffi.IG_OPT_PSELL_PAIRS_ROWS, 0)
    try:
        h = MgHierarchy(d3_case)
    finally:
        lib.ig_set_option(_ffi.IG_OPT_PSELL_LINES2, 1)
        lib.ig_set_option(_ffi.IG_OPT_PSELL_MULTI, 1)
        lib.ig_set_option(_ffi.IG_OPT_PSELL_ROWS4, 1)
        lib.ig_set_option(_ffi.IG_OPT_PSELL_ROWS4_ROWS, 1000000)
        lib.ig_set_option(_ffi.IG_OPT_PSELL_EDGE_ROWS, 100000)
        lib.ig_set_option(_ffi.IG_OPT_SMALL_ROWS, 12000)
        lib.ig_set_option(_ffi.IG_OPT_PSELL_PAIRS_ROWS, 100000)
    try:
        for l in range(1, h.levels()):
            A, _ = h.level(l)
            x = rng_vec(370 + l, A.cols())
            y0 = rng_vec(380 + l, A.rows())
            assert np.array_equal(h.spmv(l, x, 0), orc.spmv(lv, l, x, 0))
            assert np.array_equal(h.spmv(l, x, 1, y0), orc.spmv(lv, l, x, 1, y0))
        x, rep = pcg(h.A, d3_case.b, h, tol=1e-8, maxit=1000)
        st, xo, ro, it, _ = orc.pcg(lv, d3_case.b, tol=1e-8, maxit=1000, mode=orc.GPU_ORDER)
        assert st == 0 and rep.iterations == it and np.array_equal(x, xo)
    finally:
        h.close()


@pytest.mark.parametrize("complex4,one_stream", [(0, 0), (1 << 30, 0), (1 << 30, 1 << 30)])
@pytest.mark.parametrize("case_name", ["c1_case", "d3_case", "star_case"])
def test_small_level_smoother_variants_bitwise(request, case_name, complex4, one_stream):
    """The additive smoother's small-level launch variants -- complex DOFs
    one lane or four lanes each (k_as_complex / k_as_complex4), with or
    without the fork / join (k_as_blocks_simple) -- forced on every level:
    smoother, V-cycles and the whole solve bit-identical to the oracle."""
    from paper_1903_10977_b200 import MgHierarchy, _ffi, pcg
    lib = _ffi.gpu()
    case = request.getfixturevalue(case_name)
    h = MgHierarchy(case)
    lv = case.levels_c()
    try:
        assert lib.ig_hier_set_option(h.handle, _ffi.IG_OPT_COMPLEX4_ROWS, complex4) == 0
        assert lib.ig_hier_set_option(h.handle, _ffi.IG_OPT_ONE_STREAM_ROWS, one_stream) == 0
        for l in range(1, h.levels()):
            r = rng_vec(57 + l, h._n[l])
            assert np.array_equal(h.smoother_apply(l, r), orc.smoother_apply(lv, l, r))
            assert np.array_equal(h.smoother_apply(l, r, 1), orc.smoother_apply(lv, l, r, 1))
        for l in range(h.levels()):
            r = rng_vec(67 + l, h._n[l])
            assert np.array_equal(h.vcycle_at(l, r), orc.vcycle_at(lv, l, r))
        x, rep = pcg(h.A, case.b, h, tol=1e-8, maxit=1000)
        st, xo, ro, it, _ = orc.pcg(lv, case.b, tol=1e-8, maxit=1000, mode=orc.GPU_ORDER)
        assert st == 0 and rep.iterations == it
        assert np.array_equal(np.array(rep.residuals), ro) and np.array_equal(x, xo)
    finally:
        h.close()


@pytest.mark.parametrize("shift", [0, 2, 4, 6])
def test_two_line_windows_with_16_byte_aligned_vectors(d3_48_case, shift):
    """FAST8 reads its windows with 32-byte loads from the 32-byte boundary
    below each column run, found from the ADDRESS of x: a device vector that is
    only 16-byte aligned (a view starting `shift` doubles into a buffer) must
    give the same bits as the oracle (ig_level_spmv_device, A x and r - A x)."""
    import ctypes as C

    import torch

    from paper_1903_10977_b200 import MgHierarchy, _ffi
    lib = _ffi.gpu()
    lv = d3_48_case.levels_c()
    for k, v in ((_ffi.IG_OPT_PSELL_ROWS4_ROWS, 0), (_ffi.IG_OPT_PSELL_PAIRS_ROWS, 0), (_ffi.IG_OPT_SMALL_ROWS, 0)):
        lib.ig_set_option(k, v)
    try:
        h = MgHierarchy(d3_48_case)
    finally:
        for k, v in ((_ffi.IG_OPT_PSELL_ROWS4_ROWS, 1000000), (_ffi.IG_OPT_PSELL_PAIRS_ROWS, 100000),
                     (_ffi.IG_OPT_SMALL_ROWS, 12000)):
            lib.ig_set_option(k, v)
    try:
        l = h.levels() - 1
        n = h._n[l]
        x = rng_vec(611, n)
        y0 = rng_vec(612, n)
        bx = torch.zeros(n + 8, dtype=torch.float64, device="cuda")
        by = torch.zeros(n + 8, dtype=torch.float64, device="cuda")
        vx, vy = bx[shift:shift + n], by[shift:shift + n]
        assert vx.data_ptr() % 16 == 0
        vp = C.c_void_p
        vx.copy_(torch.from_numpy(x))
        torch.cuda.synchronize()
        assert lib.ig_level_spmv_device(h.handle, l, vp(vx.data_ptr()), vp(vy.data_ptr()), 0) == _ffi.IG_OK
        torch.cuda.synchronize()
        assert np.array_equal(vy.cpu().numpy(), orc.spmv(lv, l, x, 0))
        vy.copy_(torch.from_numpy(y0))
        torch.cuda.synchronize()
        assert lib.ig_level_spmv_device(h.handle, l, vp(vx.data_ptr()), vp(vy.data_ptr()), 1) == _ffi.IG_OK
        torch.cuda.synchronize()
        assert np.array_equal(vy.cpu().numpy(), orc.spmv(lv, l, x, 1, y0))
    finally:
        h.close()
