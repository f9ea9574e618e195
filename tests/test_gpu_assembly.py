"""Global assembly on the device (csrc/assemble.cuh):
from the host's element tables, ig_assemble must reproduce the host-assembled
operator and right-hand side BIT FOR BIT (assembly.cpp:164-180: setFromTriplets
summation in element order, exact zeros dropped, A = 0.5 (A + A^T))."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _check(case):
    from paper_1903_10977_b200 import assemble_on_device
    A, b, (wall, dev) = assemble_on_device(case)
    H = case.A
    assert A.shape == H.shape
    assert np.array_equal(A.row_ptr, np.asarray(H.row_ptr))
    assert np.array_equal(A.col_idx, np.asarray(H.col_idx))
    assert np.array_equal(A.val.view(np.uint64), np.asarray(H.val).view(np.uint64))
    assert np.array_equal(b.view(np.uint64), case.b.view(np.uint64))
    return wall, dev


@pytest.mark.parametrize("case_name", ["c1_case", "d3_case", "star_case"])
def test_assembly_bitwise(request, case_name):
    _check(request.getfixturevalue(case_name))


def test_assembly_box_sides_and_degree_4():
    """2D Dirichlet on the box sides (individually integrated side elements) and p = 4."""
    from paper_1903_10977_b200 import CaseConfig, SmootherConfig, build_case, configs
    _check(build_case(CaseConfig(geometry=configs.c3_geometry(1, holes=8), resolution=(64, 64, 1), degree=2,
                                 levels=3, dirichlet_box_sides=True, smoother=SmootherConfig("additive-schwarz"))))
    cfg = configs.c2(p=4, seed=configs.c2_seed())
    cfg.resolution, cfg.levels = (64, 64, 1), 3
    _check(build_case(cfg))


def test_assembly_c4_full_size():
    from paper_1903_10977_b200 import build_case, configs
    case = build_case(configs.c4())
    wall, dev = _check(case)
    print(f"C4 device assembly: {dev * 1e3:.1f} ms device, {wall:.2f} s wall; host assemble "
          f"{case.info.seconds_assemble:.2f} s (incl. cut-cell quadrature)")


@pytest.mark.parametrize("full", [False, True])
def test_assembly_thb_bitwise(full):
    """THB (C5's space): every element integrated on the device (truncated
    extraction rows, the 2D quadrature rules) and gathered per DOF over its
    support in element order -- A and b bit-identical to the host's
    assemble_g (host/thb.cpp)."""
    from paper_1903_10977_b200 import assemble_on_device, build_case, configs
    case = build_case(configs.c5() if full else configs.c5(base=32, levels=3))
    A, b, (wall, dev) = assemble_on_device(case)
    assert np.array_equal(A.row_ptr, case.A.row_ptr) and np.array_equal(A.col_idx, case.A.col_idx)
    assert np.array_equal(A.val, case.A.val) and np.array_equal(b, case.b)
    print(f"THB n={case.n}: {dev * 1e3:.1f} ms device, {wall:.2f} s wall")
