"""The host part of the device setup pipeline (igh_build_geometry): the
geometric half of build_case + MgHierarchy::build (runner.cpp:523-532,
multigrid.cpp:12-75).  Its restrictions, pre-filter Schwarz layouts,
colours, damping, level sizes and Inside-class element tables must be exactly
the full host build's -- the device then forms everything numeric from them
(tests/test_gpu_device_setup.py)."""
import ctypes as C

import numpy as np
import pytest

from paper_1903_10977_b200 import CaseConfig, MgHierarchy, SmootherConfig, _ffi, build_case, configs


def _cases():
    return {
        "c1": configs.c1(),
        "d3": configs.c4(res=16, levels=3),
        "c5s": configs.c5(base=32, levels=3),
        "ms2d": CaseConfig(geometry="disc(0.5, 0.5, 0.37)", dim=2, resolution=(32, 32, 1), degree=2, levels=3,
                           smoother=SmootherConfig("multiplicative-schwarz")),
    }


@pytest.mark.parametrize("name", list(_cases()))
def test_geometry_matches_full_build(name):
    cfg = _cases()[name]
    full = build_case(cfg)
    geo = build_case(cfg, geometry_only=True)
    try:
        assert geo.geometry_only and geo.A is None and geo.b is None
        assert geo.n_levels == full.n_levels and geo.level_dofs() == full.level_dofs()
        assert geo.n == full.n
        for l in range(1, full.n_levels):
            Rg, Rf = geo.level_R(l), full.level_R(l)
            assert Rg.shape == Rf.shape
            assert np.array_equal(Rg.row_ptr, Rf.row_ptr) and np.array_equal(Rg.col_idx, Rf.col_idx)
            assert np.array_equal(Rg.val.view(np.uint64), Rf.val.view(np.uint64))
            for a, b in zip(geo.prefilter_blocks(l), full.prefilter_blocks(l)):
                assert np.array_equal(a, b)
            assert geo.gamma(l) == full.gamma(l)
            cg, cf = geo.colors(l), full.colors(l)
            assert (cg is None) == (cf is None)
            if cg is not None:
                assert cg[1] == cf[1] and np.array_equal(cg[0], cf[0])
            assert geo.level_A(l).nnz == 0  # no operators on the geometric side
        if cfg.family != "thb":  # element tables: Inside classes equal, the individually integrated ones zero
            pg, pf = _ffi.ig_assembly(), _ffi.ig_assembly()
            assert _ffi.host().igh_assembly_payload(geo._h, C.byref(pg)) == 0
            assert _ffi.host().igh_assembly_payload(full._h, C.byref(pf)) == 0
            assert pg.n_tables == pf.n_tables and pg.n_elements == pf.n_elements
            nl = (pf.p + 1) ** pf.dim
            et = np.ctypeslib.as_array(pf.el_table, (pf.n_elements,))
            assert np.array_equal(np.ctypeslib.as_array(pg.el_table, (pg.n_elements,)), et)
            Kg = np.ctypeslib.as_array(pg.K, (pg.n_tables * nl * nl,)).reshape(pg.n_tables, -1)
            Kf = np.ctypeslib.as_array(pf.K, (pf.n_tables * nl * nl,)).reshape(pf.n_tables, -1)
            zeroed = 0
            for t in range(pf.n_tables):
                if np.any(Kg[t]):  # an Inside class: the host table itself
                    assert np.array_equal(Kg[t].view(np.uint64), Kf[t].view(np.uint64)), t
                elif np.any(Kf[t]):  # an individually integrated element: left to the device
                    zeroed += 1
            assert zeroed >= full.info.cut_elements > 0
            assert np.any(Kg)  # the Inside classes are there
        with pytest.raises(ValueError):
            MgHierarchy(geo)
        with pytest.raises(Exception):
            geo.support_fraction()
    finally:
        geo.close()
        full.close()


def test_geometry_only_write_refused(tmp_path):
    geo = build_case(configs.c1(), geometry_only=True)
    try:
        with pytest.raises(Exception):
            geo.write(str(tmp_path / "g.igh"))
    finally:
        geo.close()
