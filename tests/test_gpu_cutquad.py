"""Cut-cell quadrature on the device ("the step before
the path"): the element matrices of the 3D cut elements -- octree bisection,
Kuhn tetrahedra clipped against psi >= 0 at bisection edge roots, collapsed
Gauss rules, the interface penalty -- computed by ig_cut_quadrature3 are
bit-identical to the host's (host/assembly.cpp element3), and the fully
device-integrated global assembly reproduces the host's A and b bit for
bit, up to the full-size C4 north-star case."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _host_tables(case):
    import ctypes as C

    from paper_1903_10977_b200 import _ffi
    pay = _ffi.ig_assembly()
    assert _ffi.host().igh_assembly_payload(case._h, C.byref(pay)) == 0
    nl = (pay.p + 1) ** pay.dim
    K = np.ctypeslib.as_array(pay.K, (pay.n_tables * nl * nl,)).reshape(pay.n_tables, nl, nl)
    F = np.ctypeslib.as_array(pay.F, (pay.n_tables * nl,)).reshape(pay.n_tables, nl)
    return K, F


def _check(case):
    from paper_1903_10977_b200 import assemble_on_device, cut_quadrature_on_device
    table, K, F, vol, sec = cut_quadrature_on_device(case)
    Kh, Fh = _host_tables(case)
    assert len(table) >= case.info.cut_elements  # 2D: cut + box-side elements
    assert np.array_equal(K, Kh[table]), np.max(np.abs(K - Kh[table]))
    assert np.array_equal(F, Fh[table])
    if K.shape[1] in (8, 27):
        assert np.all((vol >= 0) & (vol <= 1 + 1e-12))
    if K.shape[1] in (8, 27):  # 3D: every table is a cut element; the min volume fraction is the host's eta
        assert vol.min() == case.info.eta
    A, b, _ = assemble_on_device(case, device_cut=True)
    assert np.array_equal(A.row_ptr, case.A.row_ptr) and np.array_equal(A.col_idx, case.A.col_idx)
    assert np.array_equal(A.val, case.A.val) and np.array_equal(b, case.b)
    return len(table), sec


def test_cut_quadrature_3d_small(d3_case):
    print(_check(d3_case))


def test_cut_quadrature_3d_depth_and_geometries():
    from paper_1903_10977_b200 import CaseConfig, SmootherConfig, build_case, configs
    for geo, depth in ((configs.c4_geometry(3), 1), (configs.c4_geometry(5), 3),
                       ("intersect(complement(sphere(0.5, 0.5, 0.5, 0.25)), box3(0.1, 0.1, 0.1, 0.9, 0.9, 0.9))", 2)):
        case = build_case(CaseConfig(geometry=geo, dim=3, resolution=(12, 12, 12), degree=2, levels=2,
                                     quad_depth=depth, dirichlet_box_sides=False,
                                     smoother=SmootherConfig("additive-schwarz")))
        print(geo, depth, _check(case))


def test_cut_quadrature_c4_full_size():
    from paper_1903_10977_b200 import build_case, configs
    n, sec = _check(build_case(configs.c4()))
    print(f"C4: {n} cut elements in {sec:.3f} s of device time")


def test_cut_quadrature_2d_small(c1_case, star_case):
    """The reference's own (2D) cut-cell quadrature: C1 (disc, box sides) and a
    Lagrange case (the star has no device level-set program: atan2 / sin, so
    it must be rejected rather than approximated)."""
    from paper_1903_10977_b200 import cut_quadrature_on_device
    print(_check(c1_case))
    with pytest.raises(NotImplementedError):
        cut_quadrature_on_device(star_case)


@pytest.mark.parametrize("p", [1, 2, 3, 4])
def test_cut_quadrature_2d_degrees(p):
    from paper_1903_10977_b200 import CaseConfig, SmootherConfig, build_case, configs
    case = build_case(CaseConfig(geometry=configs.disc_geometry(2), resolution=(24, 24, 1), degree=p, levels=2,
                                 smoother=SmootherConfig("additive-schwarz")))
    print(p, _check(case))


def test_cut_quadrature_2d_full_size():
    """C2 (p = 2, the eta < 1e-4 seed) and C3 (64 holes, Dirichlet box sides) at full size."""
    from paper_1903_10977_b200 import build_case, configs
    for cfg in (configs.c2(p=2, seed=configs.c2_seed()), configs.c3()):
        n, sec = _check(build_case(cfg))
        print(f"{n} elements in {sec:.3f} s of device time")
