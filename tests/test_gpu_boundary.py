"""Boundary semantics of the drop-in surface (include/ig_gpu.h,
paper_1903_10977_b200/__init__.py) against the reference's interface
(proj/include/immergrid/solvers.hpp:51-59, multigrid.hpp:34-75):

  * pcg / richardson multiply by the `a` they are given in the reference
    (solvers.cpp:45); the device solve uses the hierarchy's finest A, so any
    other operator must be rejected, an identical copy accepted;
  * device-built hierarchies report coarse_rank like host-built ones;
  * options are per handle (snapshot at creation, runtime options per handle);
  * unaligned device vectors are rejected instead of faulting the context.
"""
import ctypes as C

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def h1(c1_case):
    from paper_1903_10977_b200 import MgHierarchy
    h = MgHierarchy(c1_case)
    yield h
    h.close()


def test_pcg_accepts_identical_copy_and_rejects_other_operator(h1, c1_case):
    from paper_1903_10977_b200 import pcg, richardson
    x0, r0 = pcg(h1.A, c1_case.b, h1, tol=1e-8)
    A = h1.A.to_scipy().copy()
    x1, r1 = pcg(A, c1_case.b, h1, tol=1e-8)  # a copy: content hash matches
    assert np.array_equal(x0, x1) and r0.residuals == r1.residuals
    B = A.copy()
    B.data[B.nnz // 2] *= 1.0 + 1e-12
    with pytest.raises(ValueError, match="differs"):
        pcg(B, c1_case.b, h1, tol=1e-8)
    with pytest.raises(ValueError, match="differs"):
        richardson(B, c1_case.b, h1, tol=1e-8)
    with pytest.raises(ValueError, match="dimension"):
        pcg(A[:-1, :-1], c1_case.b[:-1], h1)


def test_device_built_hierarchy_reports_coarse_rank(c1_case, d3_case):
    from paper_1903_10977_b200 import MgHierarchy
    for case in (c1_case, d3_case):
        hd = MgHierarchy.build_on_device(case)
        try:
            assert hd.coarse_rank() == case.info.coarse_rank == hd.info.coarse_rank
            assert hd.info.coarse_n == case.level_dofs()[0]
        finally:
            hd.close()


def test_options_are_per_handle(c1_case):
    from paper_1903_10977_b200 import MgHierarchy, _ffi, pcg
    lib = _ffi.gpu()
    lib.ig_set_option(_ffi.IG_OPT_USE_GRAPH, 0)
    lib.ig_set_option(_ffi.IG_OPT_PSELL, 0)
    try:
        ha = MgHierarchy(c1_case)  # host-loop launches, no pattern SELL
    finally:
        lib.ig_set_option(_ffi.IG_OPT_USE_GRAPH, 1)
        lib.ig_set_option(_ffi.IG_OPT_PSELL, 1)
    hb = MgHierarchy(c1_case)  # defaults
    try:
        xa, ra = pcg(ha.A, c1_case.b, ha, tol=1e-8)  # still the handle's own (host-loop) options
        xb, rb = pcg(hb.A, c1_case.b, hb, tol=1e-8)
        assert np.array_equal(xa, xb) and ra.residuals == rb.residuals
        # runtime options of one handle
        assert lib.ig_hier_set_option(hb.handle, _ffi.IG_OPT_PDL, 0) == _ffi.IG_OK
        assert lib.ig_hier_set_option(hb.handle, _ffi.IG_OPT_USE_GRAPH, 0) == _ffi.IG_OK
        xc, rc = pcg(hb.A, c1_case.b, hb, tol=1e-8)
        assert np.array_equal(xb, xc) and rb.residuals == rc.residuals
        assert lib.ig_hier_set_option(hb.handle, _ffi.IG_OPT_USE_GRAPH, 1) == _ffi.IG_OK
        xd, rd = pcg(hb.A, c1_case.b, hb, tol=1e-8)  # graphs re-captured without PDL
        assert np.array_equal(xb, xd)
        # layout options only act at creation
        assert lib.ig_hier_set_option(hb.handle, _ffi.IG_OPT_PSELL, 0) == _ffi.IG_INVALID_ARGUMENT
    finally:
        ha.close()
        hb.close()


def test_unaligned_device_vectors_rejected(h1):
    import torch

    from paper_1903_10977_b200 import _ffi
    lib = _ffi.gpu()
    n = h1.A.rows()
    buf = torch.zeros(n + 1, dtype=torch.float64, device="cuda")
    out = torch.zeros(n + 1, dtype=torch.float64, device="cuda")
    vp = C.c_void_p
    assert lib.ig_vcycle_device(h1.handle, vp(buf[1:].data_ptr()), vp(out[:n].data_ptr())) == _ffi.IG_INVALID_ARGUMENT
    assert lib.ig_level_spmv_device(h1.handle, h1.levels() - 1, vp(buf[1:].data_ptr()), vp(out.data_ptr()), 0) \
        == _ffi.IG_INVALID_ARGUMENT
    assert lib.ig_pcg_device(h1.handle, vp(buf[1:].data_ptr()), 1e-8, 100, vp(out.data_ptr())) == _ffi.IG_INVALID_ARGUMENT
    # the context is intact: an aligned call still works
    r = torch.from_numpy(np.ones(n)).cuda()
    z = torch.empty_like(r)
    torch.cuda.synchronize()
    assert lib.ig_vcycle_device(h1.handle, vp(r.data_ptr()), vp(z.data_ptr())) == _ffi.IG_OK
    torch.cuda.synchronize()
    assert np.array_equal(z.cpu().numpy(), h1.apply(np.ones(n)))
