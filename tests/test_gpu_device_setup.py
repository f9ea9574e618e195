"""The device setup pipeline (setup_on_device):
host geometry only (igh_build_geometry), then on the GPU the cut / box-side
element quadrature (or every THB element), the row-gather assembly, the
Galerkin chain, the block factorisations, the coarsest pivoted Cholesky and
the layouts.  The finest A and b must be bit-identical to the host pipeline's
(build_case: runner.cpp:523-532 + assembly.cpp:164-180) and the solve through
the device-built hierarchy bit-identical to the host-built one's (x,
iterations, residual history) -- on small cases and on the BASELINE configs
at full size."""
import dataclasses

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _same(a, b):
    return np.array_equal(np.asarray(a).view(np.uint64), np.asarray(b).view(np.uint64))


def _check(cfg):
    from paper_1903_10977_b200 import MgHierarchy, build_case, pcg, setup_on_device
    ds = setup_on_device(cfg)
    host = build_case(cfg)
    hh = MgHierarchy(host)
    try:
        A, Ah = ds.A, host.A
        assert A.shape == Ah.shape and A.nnz == Ah.nnz
        assert np.array_equal(A.row_ptr, Ah.row_ptr) and np.array_equal(A.col_idx, Ah.col_idx)
        assert _same(A.val, Ah.val)
        assert _same(ds.b, host.b)
        assert ds.hierarchy.levels() == hh.levels()
        x, rep = pcg(ds.hierarchy.A, ds.b, ds.hierarchy, tol=1e-8, maxit=1000)
        xh, reph = pcg(hh.A, host.b, hh, tol=1e-8, maxit=1000)
        assert rep.converged and rep.iterations == reph.iterations
        assert _same(rep.residuals, reph.residuals)
        assert _same(x, xh)
        return ds.seconds, host.info.seconds_assemble + host.info.seconds_mg_setup, rep.iterations
    finally:
        hh.close()
        host.close()
        ds.close()


def _small():
    from paper_1903_10977_b200 import CaseConfig, SmootherConfig, configs
    return {
        "c1": configs.c1(),
        "d3": configs.c4(res=16, levels=3),
        "c5s": configs.c5(base=32, levels=3),
        "ms2d": CaseConfig(geometry="disc(0.5, 0.5, 0.37)", dim=2, resolution=(32, 32, 1), degree=2, levels=3,
                           smoother=SmootherConfig("multiplicative-schwarz")),
        "lag2d": CaseConfig(geometry="disc(0.5, 0.5, 0.37)", dim=2, resolution=(16, 16, 1), family="lagrange",
                            degree=2, levels=2),
        "d3p1": dataclasses.replace(configs.c4(res=16, levels=2), degree=1),
    }


@pytest.mark.parametrize("name", ["c1", "d3", "c5s", "ms2d", "lag2d", "d3p1"])
def test_device_setup_small(name):
    print(name, _check(_small()[name]))


def test_device_setup_unsupported():
    """Level sets without a device program, and 3D p = 3 (the device cut
    quadrature's shared-memory basis tables hold p <= 2), fail loudly: no
    host fallback."""
    from paper_1903_10977_b200 import CaseConfig, configs, setup_on_device
    cfg = CaseConfig(geometry="star(0.037, 0.011, 0.5, 0.1, 5)", dim=2, origin=(-1, -1, 0), extent=(2, 2, 1),
                     resolution=(16, 16, 1), family="lagrange", degree=2, levels=2)
    with pytest.raises(NotImplementedError):
        setup_on_device(cfg)
    with pytest.raises(NotImplementedError):
        setup_on_device(dataclasses.replace(configs.c4(res=16, levels=2), degree=3))


@pytest.mark.parametrize("cfg", ["c2", "c3", "c4", "c5"])
def test_device_setup_full_size(cfg):
    from paper_1903_10977_b200 import configs
    make = {"c2": lambda: configs.c2(p=2, seed=configs.c2_seed()), "c3": configs.c3, "c4": configs.c4,
            "c5": configs.c5}[cfg]
    print(cfg, _check(make()))
