"""Device-side Galerkin products (csrc/galerkin.cuh):
A_{l-1} = R_l (A_l R_l^T) computed level by level on the GPU from the finest
operator and the restrictions must reproduce the host hierarchy's coarse
operators BIT FOR BIT (row pointers, columns, value bits) -- the host products
restate Eigen's sparse-product order (MgHierarchy::build,
proj/src/multigrid.cpp:37-41), which the device keeps per entry."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _same(a, b):
    return (a.shape == b.shape and np.array_equal(np.asarray(a.row_ptr), np.asarray(b.row_ptr))
            and np.array_equal(np.asarray(a.col_idx), np.asarray(b.col_idx))
            and np.array_equal(np.asarray(a.val).view(np.uint64), np.asarray(b.val).view(np.uint64)))


def _check(case):
    from paper_1903_10977_b200 import galerkin_hierarchy
    L = case.n_levels
    R = [None] + [case.level_R(l) for l in range(1, L)]
    out, (wall, dev) = galerkin_hierarchy(case.level_A(L - 1), R)
    assert len(out) == L - 1
    for l in range(L - 1):
        assert _same(out[l], case.level_A(l)), f"level {l}"
    assert wall > 0 and dev > 0
    return wall, dev


@pytest.mark.parametrize("case_name", ["c1_case", "d3_case", "star_case"])
def test_galerkin_bitwise(request, case_name):
    _check(request.getfixturevalue(case_name))


def test_galerkin_thb_bitwise():
    """THB restriction (cross-level rows, C5 at full size)."""
    from paper_1903_10977_b200 import build_case, configs
    _check(build_case(configs.c5()))


def test_galerkin_c4_full_size():
    """The north-star hierarchy: 1,999,453-row finest operator (240 M nonzeros)."""
    from paper_1903_10977_b200 import build_case, configs
    case = build_case(configs.c4())
    wall, dev = _check(case)
    print(f"C4 device Galerkin: {dev * 1e3:.1f} ms device, {wall:.2f} s wall; host "
          f"mg setup {case.info.seconds_mg_setup:.2f} s")


def test_galerkin_rejects_mismatched_restriction(c1_case):
    from paper_1903_10977_b200 import galerkin_hierarchy
    L = c1_case.n_levels
    R = [None] + [c1_case.level_R(l) for l in range(1, L)]
    R[1], R[2] = R[2], R[1]
    with pytest.raises(ValueError):
        galerkin_hierarchy(c1_case.level_A(L - 1), R)


@pytest.mark.parametrize("short", [0, 1])
def test_galerkin_kernel_paths_bitwise(d3_case, short):
    """Both SpGEMM paths (the prefetching short-B-row kernel and the general
    one, IG_OPT_GAL_SHORT) give the host's coarse operators bit for bit."""
    from paper_1903_10977_b200 import _ffi
    lib = _ffi.gpu()
    lib.ig_set_option(_ffi.IG_OPT_GAL_SHORT, short)
    try:
        _check(d3_case)
    finally:
        lib.ig_set_option(_ffi.IG_OPT_GAL_SHORT, 1)
