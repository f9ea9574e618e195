"""B200-native solve phase of the immersed-FE / isogeometric multigrid method
(arXiv 1903.10977), behind the reference's solver/preconditioner interface.

Python mirror of the reference surface (/root/reference/proj/include/immergrid):

=========================  ===========================================================
this module                reference
=========================  ===========================================================
``pcg``                    ``pcg(A, b, precond, tol, maxit)``  solvers.hpp:51-53
``ConvergenceReport``      solvers.hpp:16-23
``Breakdown``              solvers.hpp:25-31
``NotConverged``           solvers.hpp:33-41
``MgHierarchy``            multigrid.hpp:34-74 (build / levels / level / vcycle_at /
                           apply / coarse_solve / coarse_rank)
``vcycle``                 multigrid.hpp:73-75 (1-based wrapper)
``SmootherConfig``         smoothers.hpp:18-22
``CaseConfig``/``build_case``  runner.cpp:523-532 + config.hpp (host setup)
=========================  ===========================================================

Host setup (trim, spaces, assembly, Galerkin hierarchy, Schwarz factors,
dpstrf) runs in ``libig_host.so`` (C++/OpenMP); every solve-phase operation
runs on the GPU in ``libig_gpu.so`` (hand-written sm_100a kernels).  There is
no CPU fallback: without the GPU library these calls raise.
"""
from __future__ import annotations

import ctypes as C
import dataclasses
import time
from typing import Optional, Sequence

import numpy as np

from . import _ffi

__all__ = [
    "ConvergenceReport", "Breakdown", "NotConverged", "ResolutionError",
    "SmootherConfig", "CaseConfig", "SpMat", "Case", "build_case",
    "MgHierarchy", "vcycle", "pcg", "seed_offsets", "setup_on_device", "DeviceSetup",
]

_dp = C.POINTER(C.c_double)
_ip = C.POINTER(C.c_int32)


# --------------------------------------------------------------- reports ---
@dataclasses.dataclass
class ConvergenceReport:
    """solvers.hpp:16-23: residuals[k] = ||r_k|| / ||b||, k = 0..iterations."""
    residuals: list = dataclasses.field(default_factory=list)
    iterations: int = 0
    converged: bool = False
    seconds: float = 0.0


class Breakdown(RuntimeError):
    """p^T A p <= 0 inside CG (solvers.hpp:25-31)."""

    def __init__(self, what: str, report: ConvergenceReport):
        super().__init__(what)
        self.report = report


class Diverged(RuntimeError):
    """Richardson residual grew for 10 consecutive steps (solvers.hpp:42-48)."""

    def __init__(self, what: str, report: ConvergenceReport):
        super().__init__(what)
        self.report = report


class NotConverged(RuntimeError):
    """Iteration budget exhausted; carries the report and the last x (solvers.hpp:33-41)."""

    def __init__(self, what: str, report: ConvergenceReport, x: np.ndarray):
        super().__init__(what)
        self.report = report
        self.x = x


class ResolutionError(RuntimeError):
    """The mesh cannot be coarsened the requested number of times (multigrid.hpp:13-16)."""


class GpuError(RuntimeError):
    pass


def _check(lib, rc: int, what: str):
    if rc == _ffi.IG_OK:
        return
    msg = lib.ig_last_error().decode() if hasattr(lib, "ig_last_error") else lib.igh_last_error().decode()
    if rc == _ffi.IG_INVALID_ARGUMENT:
        if "coarsenings" in msg:
            raise ResolutionError(msg)
        raise ValueError(f"{what}: {msg}")
    if rc == _ffi.IG_UNSUPPORTED:
        raise NotImplementedError(f"{what}: {msg}")
    raise GpuError(f"{what}: {msg} (status {rc})")


# ------------------------------------------------------------ host setup ---
@dataclasses.dataclass
class SmootherConfig:
    """smoothers.hpp:18-22.  Additive and multiplicative Schwarz run on the device."""
    kind: str = "additive-schwarz"
    gamma: float = 0.0          # 0 = automatic 1/max N_K
    filter_ratio: float = 1e-16


_KINDS = {"jacobi": 0, "gauss-seidel": 1, "additive-schwarz": 2, "multiplicative-schwarz": 3}


@dataclasses.dataclass
class CaseConfig:
    """Case description (the subset of config.hpp:34-86 the solve needs, plus 3D)."""
    geometry: str = "constant(1)"
    dim: int = 2
    origin: Sequence[float] = (0.0, 0.0, 0.0)
    extent: Sequence[float] = (1.0, 1.0, 1.0)
    resolution: Sequence[int] = (16, 16, 16)
    family: str = "bspline"     # "bspline" | "lagrange" (2D)
    degree: int = 2
    levels: int = 2
    quad_depth: int = 3
    gauss_order: int = 0         # 0 = p + 1
    classify_depth: int = 2
    edge_tol: float = 1e-12
    body_force: float = 1.0
    beta: float = 0.0            # 0 = 2/h
    dirichlet_box_sides: bool = True
    smoother: SmootherConfig = dataclasses.field(default_factory=SmootherConfig)
    threads: int = 0
    # THB local refinement (family="thb", 2D): refine-by-box passes, then
    # `refine_passes` passes near the circle (cx, cy, r) within refine_dist.
    refine_boxes: Sequence[Sequence[float]] = ()
    refine_passes: int = 0
    refine_circle: Sequence[float] = (0.0, 0.0, 0.0)
    refine_dist: float = 0.0

    def to_c(self) -> _ffi.igh_config:
        c = _ffi.igh_config()
        _ffi.host().igh_config_default(C.byref(c))
        self._geo = self.geometry.encode()
        c.dim = self.dim
        c.geometry = self._geo
        for i in range(3):
            c.origin[i] = float(self.origin[i]) if i < len(self.origin) else 0.0
            c.extent[i] = float(self.extent[i]) if i < len(self.extent) else 1.0
            c.resolution[i] = int(self.resolution[i]) if i < len(self.resolution) else 1
        fam = self.family.lower()
        c.family = 0 if fam.startswith("lag") else (2 if fam == "thb" else 1)
        self._boxes = np.ascontiguousarray(np.array(self.refine_boxes, dtype=np.float64).reshape(-1))
        c.n_refine_boxes = len(self.refine_boxes)
        c.refine_boxes = self._boxes.ctypes.data_as(_dp) if len(self.refine_boxes) else None
        c.refine_passes = self.refine_passes
        for i in range(3):
            c.refine_circle[i] = float(self.refine_circle[i])
        c.refine_dist = self.refine_dist
        c.degree = self.degree
        c.levels = self.levels
        c.quad_depth = self.quad_depth
        c.gauss_order = self.gauss_order
        c.classify_depth = self.classify_depth
        c.edge_tol = self.edge_tol
        c.body_force = self.body_force
        c.beta = self.beta
        c.dirichlet_box_sides = 1 if self.dirichlet_box_sides else 0
        c.smoother_kind = _KINDS[self.smoother.kind]
        c.gamma = self.smoother.gamma
        c.filter_ratio = self.smoother.filter_ratio
        c.threads = self.threads
        return c


def seed_offsets(seed: int = 1, count: int = 3):
    """delta = Rng(seed).uniform(-0.01, 0.01) x count (common.hpp:43-58)."""
    m = (1 << 64) - 1
    s = seed
    out = []
    for _ in range(count):
        s = (s + 0x9E3779B97F4A7C15) & m
        z = s
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & m
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & m
        z ^= z >> 31
        u = (z >> 11) * 2.0 ** -53
        out.append(-0.01 + 0.02 * u)
    return out


class SpMat:
    """CSR view (== Eigen RowMajor compressed, int32 indices)."""

    def __init__(self, n_rows, n_cols, row_ptr, col_idx, val, _owner=None):
        self.shape = (int(n_rows), int(n_cols))
        self.row_ptr = row_ptr
        self.col_idx = col_idx
        self.val = val
        self._owner = _owner

    @classmethod
    def from_c(cls, m: _ffi.ig_csr, owner=None) -> "SpMat":
        nr, nc, nnz = m.n_rows, m.n_cols, m.nnz
        if nr == 0:
            return cls(0, nc, np.zeros(1, np.int32), np.zeros(0, np.int32), np.zeros(0), owner)
        rp = np.ctypeslib.as_array(m.row_ptr, (nr + 1,))
        ci = np.ctypeslib.as_array(m.col_idx, (nnz,)) if nnz else np.zeros(0, np.int32)
        vv = np.ctypeslib.as_array(m.val, (nnz,)) if nnz else np.zeros(0)
        return cls(nr, nc, rp, ci, vv, owner)

    @property
    def nnz(self) -> int:
        return int(self.col_idx.shape[0])

    def rows(self) -> int:
        return self.shape[0]

    def cols(self) -> int:
        return self.shape[1]

    def to_scipy(self):
        import scipy.sparse as sp
        return sp.csr_matrix((self.val, self.col_idx, self.row_ptr), shape=self.shape)


def galerkin_hierarchy(A_fine: "SpMat", R: Sequence[Optional["SpMat"]]):
    """Device-side Galerkin products of MgHierarchy::build
    (proj/src/multigrid.cpp:37-41, `r * (A * r.transpose())` level by level):
    A_{l-1} = R_l (A_l R_l^T) for l = L-1 .. 1 on the GPU, bit-identical to the
    host (Eigen-order) products.  `R[l]` is level l's restriction (R[0] unused).
    Returns ([A_0 .. A_{L-2}] as SpMat with numpy-owned arrays,
    (wall_seconds, device_seconds))."""
    lib = _ffi.gpu()
    L = len(R)

    keep = []  # arrays referenced by the C structs stay alive until the call returns

    def to_c(m: SpMat):
        rp = np.ascontiguousarray(m.row_ptr, np.int32)
        ci = np.ascontiguousarray(m.col_idx, np.int32)
        vv = np.ascontiguousarray(m.val, np.float64)
        keep.extend((rp, ci, vv))
        return _ffi.ig_csr(m.shape[0], m.shape[1], m.nnz, rp.ctypes.data_as(C.POINTER(C.c_int32)),
                           ci.ctypes.data_as(C.POINTER(C.c_int32)), vv.ctypes.data_as(C.POINTER(C.c_double)))

    a = to_c(A_fine)
    rs = (_ffi.ig_csr * L)()
    for l in range(1, L):
        rs[l] = to_c(R[l])
    out = (_ffi.ig_csr * max(L - 1, 1))()
    sec = (C.c_double * 2)()
    _check(lib, lib.ig_galerkin_hierarchy(C.byref(a), rs, L, out, sec), "ig_galerkin_hierarchy")
    res = []
    try:
        for l in range(L - 1):
            m = SpMat.from_c(out[l])
            res.append(SpMat(m.shape[0], m.shape[1], m.row_ptr.copy(), m.col_idx.copy(), m.val.copy()))
    finally:
        for l in range(L - 1):
            lib.ig_csr_free(C.byref(out[l]))
    del keep
    return res, (sec[0], sec[1])


def factorize_blocks(A: "SpMat", blk_ptr, blk_dofs, filter_ratio: float = 1e-16):
    """Device batched Schwarz block factorisation (make_smoother's
    factorize_blocks, proj/src/smoothers.cpp:131-162): eigen-filter + LLT of
    every pre-filter block.  Returns (blk_ptr, blk_dofs, fac_ptr, fac,
    filtered_dofs, (wall_seconds, device_seconds)) of the post-filter layout,
    bit-identical to the host factorisation."""
    lib = _ffi.gpu()
    rp = np.ascontiguousarray(A.row_ptr, np.int32)
    ci = np.ascontiguousarray(A.col_idx, np.int32)
    vv = np.ascontiguousarray(A.val, np.float64)
    a = _ffi.ig_csr(A.shape[0], A.shape[1], A.nnz, rp.ctypes.data_as(C.POINTER(C.c_int32)),
                    ci.ctypes.data_as(C.POINTER(C.c_int32)), vv.ctypes.data_as(C.POINTER(C.c_double)))
    bp = np.ascontiguousarray(blk_ptr, np.int32)
    bd = np.ascontiguousarray(blk_dofs, np.int32)
    nb = bp.shape[0] - 1
    out = _ffi.ig_blocks()
    filt = C.c_int64()
    sec = (C.c_double * 2)()
    _check(lib, lib.ig_factorize_blocks(C.byref(a), nb, bp.ctypes.data_as(C.POINTER(C.c_int32)),
                                        bd.ctypes.data_as(C.POINTER(C.c_int32)), float(filter_ratio),
                                        C.byref(out), C.byref(filt), sec), "ig_factorize_blocks")
    try:
        optr = np.ctypeslib.as_array(out.blk_ptr, (nb + 1,)).copy()
        odofs = np.ctypeslib.as_array(out.blk_dofs, (max(int(optr[-1]), 1),))[:int(optr[-1])].copy()
        ofp = np.ctypeslib.as_array(out.fac_ptr, (nb + 1,)).copy()
        ofac = np.ctypeslib.as_array(out.fac, (max(int(ofp[-1]), 1),))[:int(ofp[-1])].copy()
    finally:
        lib.ig_blocks_free(C.byref(out))
    return optr, odofs, ofp, ofac, int(filt.value), (sec[0], sec[1])


def cut_quadrature_on_device(case):
    """Element matrices of the finest level's individually integrated
    elements computed on the device: 3D cut elements (ig_cut_quadrature3:
    octree + clipped Kuhn tetrahedra + interface triangles) or, in 2D, cut
    and box-side elements (ig_cut_quadrature2: the reference's recurse_cut /
    leaf polygons / chord refinement / fan triangulation / interface and side
    rules) -- the host's element integration operation for operation.
    Returns (table, K, F, vol, seconds): `table[k]` is the element-table index
    the host stored the same element under (igh_assembly_payload), K is
    n x nl x nl, F n x nl.  Uniform B-spline / Lagrange cases."""
    lib = _ffi.gpu()
    if _ffi.host().igh_cut3_payload(case._h, C.byref(_ffi.ig_cut3())) != _ffi.IG_OK:  # 2D (or unsupported)
        pay = _ffi.ig_cut2()
        _check(_ffi.host(), _ffi.host().igh_cut2_payload(case._h, C.byref(pay)), "igh_cut2_payload")
        n, nl, fn = pay.n_elem, (pay.p + 1) ** 2, lib.ig_cut_quadrature2
    else:
        pay = _ffi.ig_cut3()
        _check(_ffi.host(), _ffi.host().igh_cut3_payload(case._h, C.byref(pay)), "igh_cut3_payload")
        n, nl, fn = pay.n_cut, (pay.p + 1) ** 3, lib.ig_cut_quadrature3
    K = np.zeros((n, nl, nl))
    F = np.zeros((n, nl))
    vol = np.zeros(n)
    sec = C.c_double()
    _check(lib, fn(C.byref(pay), K.ctypes.data_as(_dp), F.ctypes.data_as(_dp), vol.ctypes.data_as(_dp),
                   C.byref(sec)), "cut quadrature")
    table = np.ctypeslib.as_array(pay.table, (n,)).copy() if n else np.zeros(0, np.int32)
    return table, K, F, vol, sec.value


def assemble_on_device(case, device_cut: bool = False):
    """The finest level's global assembly on the GPU:
    the element tables go through ig_assemble, which sums the element
    contributions in the reference's setFromTriplets order and symmetrises
    (assembly.cpp:164-180).  device_cut: the individually integrated
    elements' tables are computed on the device too (cut_quadrature_on_device),
    else the host case's tables are used.  THB cases: every element is
    integrated and gathered on the device (ig_assemble_thb).  Returns (A as SpMat, b,
    (wall_seconds, device_seconds)), bit-identical to the host assembly
    (case.A, case.b)."""
    lib = _ffi.gpu()
    thb = _ffi.ig_thb_asm()
    if _ffi.host().igh_thb_payload(case._h, C.byref(thb)) == _ffi.IG_OK:  # THB: element integration + gather
        out = _ffi.ig_csr()
        b = np.empty(thb.n)
        sec = (C.c_double * 2)()
        _check(lib, lib.ig_assemble_thb(C.byref(thb), C.byref(out), b.ctypes.data_as(_dp), sec), "ig_assemble_thb")
        try:
            m = SpMat.from_c(out)
            A = SpMat(m.shape[0], m.shape[1], m.row_ptr.copy(), m.col_idx.copy(), m.val.copy())
        finally:
            lib.ig_csr_free(C.byref(out))
        return A, b, (sec[0], sec[1])
    pay = _ffi.ig_assembly()
    _check(_ffi.host(), _ffi.host().igh_assembly_payload(case._h, C.byref(pay)), "igh_assembly_payload")
    keep = None
    if device_cut:
        table, Kc, Fc, _, _ = cut_quadrature_on_device(case)
        q = pay.p + 1
        nl = q ** pay.dim
        Kall = np.ctypeslib.as_array(pay.K, (pay.n_tables * nl * nl,)).reshape(pay.n_tables, nl * nl).copy()
        Fall = np.ctypeslib.as_array(pay.F, (pay.n_tables * nl,)).reshape(pay.n_tables, nl).copy()
        Kall[table] = Kc.reshape(len(table), nl * nl)
        Fall[table] = Fc
        keep = (Kall, Fall)
        pay.K = Kall.ctypes.data_as(_dp)
        pay.F = Fall.ctypes.data_as(_dp)
    out = _ffi.ig_csr()
    b = np.empty(pay.n)
    sec = (C.c_double * 2)()
    _check(lib, lib.ig_assemble(C.byref(pay), C.byref(out), b.ctypes.data_as(C.POINTER(C.c_double)), sec),
           "ig_assemble")
    try:
        m = SpMat.from_c(out)
        A = SpMat(m.shape[0], m.shape[1], m.row_ptr.copy(), m.col_idx.copy(), m.val.copy())
    finally:
        lib.ig_csr_free(C.byref(out))
    del keep
    return A, b, (sec[0], sec[1])


@dataclasses.dataclass
class DeviceSetup:
    """setup_on_device's result: the geometry-only host case, the device-
    assembled finest system (A, b) and the device-built hierarchy."""
    case: "Case"
    A: "SpMat"
    b: np.ndarray
    hierarchy: "MgHierarchy"
    seconds: dict

    def close(self):
        self.hierarchy.close()
        self.case.close()


def setup_on_device(cfg_or_case) -> DeviceSetup:
    """The whole setup with every numeric stage on the GPU (SURVEY.md 8(f)
    rows 2-3; runner.cpp:523-532 build_case + multigrid.cpp:12-75 build):
      host    igh_build_geometry: trimmed spaces, restrictions, pre-filter
              Schwarz layouts, Inside-class element tables (no integration of
              cut / box-side elements, no assembly, no Galerkin, no factors);
      device  cut-element quadrature (ig_cut_quadrature2/3) or, for THB, every
              element's integration (ig_assemble_thb), then the row-gather
              assembly + symmetrisation (ig_assemble);
      device  Galerkin chain, block eigen-filter + LLT, coarsest pivoted
              Cholesky, layouts (ig_hier_build).
    A, b and the hierarchy are bit-identical to the host pipeline's
    (build_case + MgHierarchy; tests/test_gpu_device_setup.py).  Level sets
    without a device program (star / affine) are IG_UNSUPPORTED.  seconds:
    host_geometry, assembly (wall; device part in assembly_device),
    hierarchy (wall; device kernels in hierarchy_device), total."""
    t0 = time.perf_counter()
    own = not isinstance(cfg_or_case, Case)
    case = build_case(cfg_or_case, geometry_only=True) if own else cfg_or_case
    try:
        if not case.geometry_only:
            raise ValueError("setup_on_device: pass a CaseConfig or a geometry-only case")
        t1 = time.perf_counter()
        A, b, asec = assemble_on_device(case, device_cut=True)
        t2 = time.perf_counter()
        h = MgHierarchy.build_on_device(case, A)
        t3 = time.perf_counter()
    except BaseException:
        if own:
            case.close()
        raise
    sec = {"host_geometry": t1 - t0, "assembly": t2 - t1, "assembly_device": asec[1],
           "hierarchy": t3 - t2, "hierarchy_device": h.setup_seconds[1], "total": t3 - t0}
    return DeviceSetup(case, A, b, h, sec)


class TooLarge(RuntimeError):
    """spectral.hpp:16 TooLarge."""


@dataclasses.dataclass
class SpectrumResult:
    """spectral.hpp:24-31."""
    eigenvalues: np.ndarray
    vectors: Optional[np.ndarray]
    lambda_min: float
    lambda_max: float
    kappa: float


def dense_spectrum(h: "MgHierarchy", name: str = "vcycle", want_vectors: bool = False,
                   dense_limit: int = 6000) -> SpectrumResult:
    """dense_spectrum of a composed operator (runner.cpp:84-122 + spectral.cpp:28-91):
    the operator is materialised column by column ON THE DEVICE
    (ig_operator_columns: A e_j, then the V-cycle / symmetric smoother), the
    dense nonsymmetric eigenproblem runs on the host (the reference calls
    LAPACK dgeev there too).  name: "vcycle" (M A), "as2" / "ms2" (the finest
    smoother's apply_symmetric(A v); must match the hierarchy's smoother kind),
    "jacobi" (D^-1 A)."""
    n = h.A.rows()
    if n < 1:
        raise ValueError("dense_spectrum: n must be positive")
    if n > dense_limit:
        raise TooLarge(f"dense_spectrum: n = {n} exceeds dense limit {dense_limit}")
    lib = _ffi.gpu()
    if name == "vcycle":
        kind = _ffi.IG_OP_VCYCLE
    elif name in ("as2", "ms2"):
        want = 2 if name == "as2" else 3
        if h.levels() < 2 or h._lv[h.levels() - 1].smoother_kind != want:
            raise ValueError(f"dense_spectrum: {name} needs a hierarchy built with that smoother")
        kind = _ffi.IG_OP_SMOOTHER_SYMMETRIC
    elif name in ("jacobi", "A"):
        kind = _ffi.IG_OP_A
    else:
        raise ValueError(f'spectrum: unknown operator "{name}" (one of: jacobi, as2, ms2, vcycle)')
    m = np.empty((n, n), order="F")
    _check(lib, lib.ig_operator_columns(h.handle, kind, 0, n, m.ctypes.data_as(C.POINTER(C.c_double))),
           "ig_operator_columns")
    if name == "jacobi":
        d = h.A.to_scipy().diagonal()
        if np.any(d <= 0.0):
            raise RuntimeError("spectrum: operator diagonal is not positive")
        m = m / d[:, None]
    if want_vectors:
        wr_c, vr = np.linalg.eig(m)
    else:
        wr_c, vr = np.linalg.eigvals(m), None
    wr, wi = wr_c.real, wr_c.imag
    scale = np.max(np.abs(wr))
    if np.max(np.abs(wi)) > 1e-8 * max(scale, 1e-300):
        raise RuntimeError("dense_spectrum: eigenvalues have imaginary parts beyond tolerance "
                           "(operator not similar to a symmetric one)")
    order = np.argsort(wr, kind="stable")
    ev = wr[order]
    vecs = vr[:, order].real if want_vectors else None
    lmax = float(ev[-1])
    cutoff = 1e-12 * abs(lmax)
    nz = ev[ev > cutoff]
    smallest = float(nz[0]) if nz.size else lmax
    return SpectrumResult(ev, vecs, float(ev[0]), lmax, lmax / smallest)


class Case:
    """Host-built case: fine system (A, b) and the multigrid hierarchy payload
    that crosses the C-ABI (owned by libig_host.so until close()).
    geometry_only (build_case(cfg, geometry_only=True), igh_build_geometry):
    spaces, restrictions, pre-filter block layouts and element tables only --
    A and b are None until the device pipeline (setup_on_device) forms them."""

    def __init__(self, handle: C.c_void_p, cfg: Optional[CaseConfig] = None, geometry_only: bool = False):
        self._h = handle
        self.config = cfg
        self.geometry_only = geometry_only
        lib = _ffi.host()
        self._lv = C.POINTER(_ffi.ig_level)()
        nl = C.c_int32()
        self._co = C.POINTER(_ffi.ig_coarse)()
        lib.igh_levels(self._h, C.byref(self._lv), C.byref(nl), C.byref(self._co))
        self.n_levels = nl.value
        info = _ffi.igh_info()
        lib.igh_get_info(self._h, C.byref(info))
        self.info = info
        if geometry_only:
            self.b = None
            self.A = None
            return
        n = C.c_int32()
        bp = lib.igh_rhs(self._h, C.byref(n))
        self.b = np.ctypeslib.as_array(bp, (n.value,)).copy()
        self.A = SpMat.from_c(self._lv[self.n_levels - 1].A, self)

    @property
    def n(self) -> int:
        return self.info.n[self.n_levels - 1]

    def level_dofs(self):
        return [self.info.n[i] for i in range(self.n_levels)]

    def levels_c(self):
        return self._lv, self.n_levels, self._co

    def level_A(self, l: int) -> SpMat:
        return SpMat.from_c(self._lv[l].A, self)

    def prefilter_blocks(self, l: int):
        """(blk_ptr, blk_dofs) of level l's pre-filter Schwarz layout (select_blocks)."""
        nb = C.c_int32()
        bp = C.POINTER(C.c_int32)()
        bd = C.POINTER(C.c_int32)()
        _check(_ffi.host(), _ffi.host().igh_prefilter_blocks(self._h, l, C.byref(nb), C.byref(bp), C.byref(bd)),
               "igh_prefilter_blocks")
        ptr = np.ctypeslib.as_array(bp, (nb.value + 1,)).copy()
        return ptr, np.ctypeslib.as_array(bd, (max(int(ptr[-1]), 1),))[:int(ptr[-1])].copy()

    def level_R(self, l: int) -> SpMat:
        return SpMat.from_c(self._lv[l].R, self)

    def gamma(self, l: int) -> float:
        return self._lv[l].gamma

    def blocks(self, l: int):
        """(blk_ptr, blk_dofs, fac_ptr, fac) of level l (post-filter)."""
        b = self._lv[l].blocks
        nb = b.n_blocks
        if nb == 0:
            return None
        ptr = np.ctypeslib.as_array(b.blk_ptr, (nb + 1,))
        dofs = np.ctypeslib.as_array(b.blk_dofs, (int(ptr[-1]),))
        fptr = np.ctypeslib.as_array(b.fac_ptr, (nb + 1,))
        fac = np.ctypeslib.as_array(b.fac, (int(fptr[-1]),))
        return ptr, dofs, fptr, fac

    def colors(self, l: int):
        """(color_of per block, n_colors) of level l (multiplicative sweeps; None otherwise)."""
        b = self._lv[l].blocks
        if b.n_colors == 0 or not b.color_of:
            return None
        return np.ctypeslib.as_array(b.color_of, (b.n_blocks,)), b.n_colors

    def coarse(self):
        co = self._co.contents
        n = co.n
        L = np.ctypeslib.as_array(co.L, (n * n,)).reshape(n, n, order="F")
        piv = np.ctypeslib.as_array(co.piv, (max(n, 1),))[:n]
        return L, piv, co.rank

    def support_fraction(self) -> np.ndarray:
        """Finest level, per DOF: physical support volume / untrimmed support
        cell volume (igh_support_fraction; uniform spaces only)."""
        out = np.zeros(self.n)
        _check(_ffi.host(), _ffi.host().igh_support_fraction(self._h, out.ctypes.data_as(C.POINTER(C.c_double))),
               "support_fraction")
        return out

    def anchors(self, l: int) -> np.ndarray:
        out = np.zeros((self.info.n[l], 3), np.int32)
        _check(_ffi.host(), _ffi.host().igh_anchors(self._h, l, out.ctypes.data_as(_ip)), "anchors")
        return out

    def write(self, path: str):
        _check(_ffi.host(), _ffi.host().igh_write(self._h, path.encode()), "igh_write")

    @classmethod
    def read(cls, path: str) -> "Case":
        h = C.c_void_p()
        _check(_ffi.host(), _ffi.host().igh_read(path.encode(), C.byref(h)), "igh_read")
        return cls(h)

    def close(self):
        if self._h:
            _ffi.host().igh_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def build_case(cfg: CaseConfig, geometry_only: bool = False) -> Case:
    """build_case + MgHierarchy::build host half (runner.cpp:523-532, multigrid.cpp:12-75).
    geometry_only: the geometric half only (igh_build_geometry) -- the host
    part of the device setup pipeline (setup_on_device)."""
    c = cfg.to_c()
    h = C.c_void_p()
    fn = _ffi.host().igh_build_geometry if geometry_only else _ffi.host().igh_build
    _check(_ffi.host(), fn(C.byref(c), C.byref(h)), "igh_build_geometry" if geometry_only else "igh_build")
    return Case(h, cfg, geometry_only)


# -------------------------------------------------------------- device -----
def _as_f64(v, n: int) -> np.ndarray:
    a = np.ascontiguousarray(v, dtype=np.float64)
    if a.shape != (n,):
        raise ValueError(f"vector of size {a.shape} where {n} is required")
    return a


class MgHierarchy:
    """Device-resident multigrid hierarchy (multigrid.hpp:34-74).  Immutable
    after build; calls on one handle serialise (the library holds a mutex)."""

    def __init__(self, case):
        """`case`: a host-built Case, or any payload exposing levels_c() ->
        (ig_level*, n_levels, ig_coarse*) (the C-ABI boundary structs)."""
        if getattr(case, "geometry_only", False):
            raise ValueError("MgHierarchy: a geometry-only case has no operators (use setup_on_device)")
        lib = _ffi.gpu()
        lv, nl, co = case.levels_c()
        self._h = C.c_void_p()
        _check(lib, lib.ig_hier_create(lv, nl, co, C.byref(self._h)), "ig_hier_create")
        self.case = case
        self._lv = lv
        self._n = [lv[i].A.n_rows for i in range(nl)]
        self.A = SpMat.from_c(lv[nl - 1].A, case)
        self._rank = co.contents.rank
        info = _ffi.ig_info()
        lib.ig_hier_info(self._h, C.byref(info))
        self.info = info

    @staticmethod
    def build_on_device(case, A: Optional["SpMat"] = None) -> "MgHierarchy":
        """MgHierarchy::build's algebraic half on the GPU (ig_hier_build): the
        Galerkin chain, the Schwarz block factorisations and the coarsest
        pivoted Cholesky are computed on the device from the finest operator,
        the restrictions and the pre-filter block layouts of the host-built
        `case` (its own coarse operators and factors are NOT used).  The
        handle is bit-identical to MgHierarchy(case).  A: the finest operator
        (default: the case's; required for a geometry-only case -- the device
        assembly's, setup_on_device).  self.setup_seconds = (wall, device
        kernels, ig_hier_create)."""
        lib = _ffi.gpu()
        lv, nl, co = case.levels_c()
        if A is None:
            if getattr(case, "geometry_only", False):
                raise ValueError("build_on_device: a geometry-only case needs the finest operator A")
            A = SpMat.from_c(lv[nl - 1].A, case)
        if A.shape != (case.n, case.n):
            raise ValueError(f"build_on_device: A is {A.shape}, the finest level has {case.n} DOFs")
        sm = case.config.smoother if case.config is not None else SmootherConfig()
        R = (_ffi.ig_csr * nl)()
        pre = (_ffi.ig_blocks * nl)()
        gam = (C.c_double * nl)()
        keep = []
        for l in range(nl):
            gam[l] = lv[l].gamma
            if l == 0:
                continue
            R[l] = lv[l].R
            bp, bd = case.prefilter_blocks(l)
            keep += [bp, bd]
            pre[l].n_blocks = bp.shape[0] - 1
            pre[l].blk_ptr = bp.ctypes.data_as(C.POINTER(C.c_int32))
            pre[l].blk_dofs = bd.ctypes.data_as(C.POINTER(C.c_int32))
            pre[l].n_colors = lv[l].blocks.n_colors
            pre[l].color_of = lv[l].blocks.color_of
        self = MgHierarchy.__new__(MgHierarchy)
        self._h = C.c_void_p()
        sec = (C.c_double * 3)()
        rp = np.ascontiguousarray(A.row_ptr, np.int32)
        ci = np.ascontiguousarray(A.col_idx, np.int32)
        vv = np.ascontiguousarray(A.val, np.float64)
        keep += [rp, ci, vv]
        a = _ffi.ig_csr(A.shape[0], A.shape[1], A.nnz, rp.ctypes.data_as(C.POINTER(C.c_int32)),
                        ci.ctypes.data_as(C.POINTER(C.c_int32)), vv.ctypes.data_as(C.POINTER(C.c_double)))
        _check(lib, lib.ig_hier_build(C.byref(a), R, pre, gam, lv[nl - 1].smoother_kind if nl > 1 else 2,
                                      float(sm.filter_ratio), nl, C.byref(self._h), sec), "ig_hier_build")
        del keep
        self.case = case
        self._lv = lv
        self._n = [lv[i].A.n_rows for i in range(nl)]
        self.A = A
        info = _ffi.ig_info()
        lib.ig_hier_info(self._h, C.byref(info))
        self.info = info
        self._rank = info.coarse_rank  # the device pstrf's rank
        self.setup_seconds = (sec[0], sec[1], sec[2])
        return self

    @staticmethod
    def build(case_or_cfg, levels: Optional[int] = None, smoother: Optional[SmootherConfig] = None) -> "MgHierarchy":
        if isinstance(case_or_cfg, CaseConfig):
            cfg = dataclasses.replace(case_or_cfg)
            if levels is not None:
                cfg.levels = levels
            if smoother is not None:
                cfg.smoother = smoother
            case_or_cfg = build_case(cfg)
        return MgHierarchy(case_or_cfg)

    def levels(self) -> int:
        return len(self._n)

    def level(self, l: int):
        return SpMat.from_c(self._lv[l].A, self.case), SpMat.from_c(self._lv[l].R, self.case)

    def coarse_rank(self) -> int:
        return self._rank

    @property
    def handle(self):
        return self._h

    def vcycle_at(self, l: int, r) -> np.ndarray:
        if not 0 <= l < self.levels():
            raise ValueError("vcycle_at: level out of range")
        rr = _as_f64(r, self._n[l])
        x = np.empty_like(rr)
        lib = _ffi.gpu()
        _check(lib, lib.ig_vcycle_at(self._h, l, rr.ctypes.data_as(_dp), x.ctypes.data_as(_dp)), "vcycle_at")
        return x

    def apply(self, r) -> np.ndarray:
        return self.vcycle_at(self.levels() - 1, r)

    __call__ = apply

    def coarse_solve(self, r) -> np.ndarray:
        return self.vcycle_at(0, r)

    def smoother_apply(self, l: int, r, direction: int = 0) -> np.ndarray:
        """Smoother::apply(r, dir) of level l: direction 0 Forward, 1 Reverse."""
        rr = _as_f64(r, self._n[l])
        x = np.empty_like(rr)
        lib = _ffi.gpu()
        _check(lib, lib.ig_smoother_apply_dir(self._h, l, rr.ctypes.data_as(_dp), x.ctypes.data_as(_dp),
                                              int(direction)), "smoother_apply")
        return x

    def smoother_apply_symmetric(self, l: int, r) -> np.ndarray:
        """Smoother::apply_symmetric (smoothers.cpp:211-214)."""
        rr = _as_f64(r, self._n[l])
        x = np.empty_like(rr)
        lib = _ffi.gpu()
        _check(lib, lib.ig_smoother_apply_symmetric(self._h, l, rr.ctypes.data_as(_dp), x.ctypes.data_as(_dp)),
               "smoother_apply_symmetric")
        return x

    def spmv(self, l: int, x, mode: int = 0, y=None) -> np.ndarray:
        """mode 0: A x, 1: y - A x, 2: R x, 3: R^T x (ig_level_spmv)."""
        A, R = self.level(l)
        nin = A.cols() if mode <= 1 else (R.cols() if mode == 2 else R.rows())
        nout = A.rows() if mode <= 1 else (R.rows() if mode == 2 else R.cols())
        xx = _as_f64(x, nin)
        yy = np.zeros(nout) if y is None else _as_f64(y, nout).copy()
        lib = _ffi.gpu()
        _check(lib, lib.ig_level_spmv(self._h, l, xx.ctypes.data_as(_dp), yy.ctypes.data_as(_dp), mode), "level_spmv")
        return yy

    def close(self):
        if getattr(self, "_h", None):
            _ffi.gpu().ig_hier_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def vcycle(h: MgHierarchy, ell: int, r) -> np.ndarray:
    """One-based level wrapper (multigrid.hpp:73-75)."""
    return h.vcycle_at(ell - 1, r)


def _check_operator(a, precond: MgHierarchy, what: str):
    """The reference multiplies by the `a` it is given (solvers.cpp:45); the
    device solve multiplies by the hierarchy's finest A.  Accept `a` only when
    it IS that operator: None, the same object, or a CSR (SpMat / scipy) with
    identical sizes, row pointers, columns and value bits (ig_hier_matches)."""
    fineA = precond.A
    if a is None or a is fineA:
        return
    shape = getattr(a, "shape", None)
    if shape is None or tuple(shape) != fineA.shape:
        raise ValueError(f"{what}: dimension mismatch")
    if isinstance(a, SpMat):
        rp, ci, vv = a.row_ptr, a.col_idx, a.val
    else:
        try:
            csr = a.tocsr()
        except AttributeError:
            raise TypeError(f"{what}: `a` must be the CSR operator the hierarchy was built on") from None
        rp, ci, vv = csr.indptr, csr.indices, csr.data
    rp = np.ascontiguousarray(rp, np.int32)
    ci = np.ascontiguousarray(ci, np.int32)
    vv = np.ascontiguousarray(vv, np.float64)
    m = _ffi.ig_csr()
    m.n_rows, m.n_cols = shape
    m.nnz = int(rp[-1])
    m.row_ptr = rp.ctypes.data_as(C.POINTER(C.c_int32))
    m.col_idx = ci.ctypes.data_as(C.POINTER(C.c_int32))
    m.val = vv.ctypes.data_as(_dp)
    lib = _ffi.gpu()
    if lib.ig_hier_matches(precond.handle, C.byref(m)) != _ffi.IG_OK:
        raise ValueError(f"{what}: {lib.ig_last_error().decode()}")


def pcg(a, b, precond: MgHierarchy, tol: float = 1e-10, maxit: int = 1000):
    """Preconditioned CG with zero initial guess (solvers.cpp:17-71), run
    entirely on the device.  ``precond`` must be the GPU MgHierarchy built on
    ``a`` (the reference passes the same fine matrix to build and pcg,
    runner.cpp:219,233).  Returns (x, ConvergenceReport); raises Breakdown /
    NotConverged like the reference."""
    if not isinstance(precond, MgHierarchy):
        raise TypeError("pcg: the preconditioner must be a device MgHierarchy (no CPU fallback)")
    fineA = precond.A
    _check_operator(a, precond, "pcg")
    n = fineA.rows()
    if fineA.rows() != fineA.cols() or np.shape(b) != (n,):
        raise ValueError("pcg: dimension mismatch")
    bb = _as_f64(b, n)
    x = np.zeros(n)
    res = np.zeros(max(maxit, 0) + 1)
    it = C.c_int32()
    sec = C.c_double()
    lib = _ffi.gpu()
    rc = lib.ig_pcg(precond.handle, bb.ctypes.data_as(_dp), float(tol), int(maxit), x.ctypes.data_as(_dp),
                    res.ctypes.data_as(_dp), C.byref(it), C.byref(sec))
    k = it.value
    rep = ConvergenceReport(residuals=res[: k + 1].tolist(), iterations=k, converged=(rc == _ffi.IG_OK),
                            seconds=sec.value)
    if rc == _ffi.IG_OK:
        return x, rep
    msg = lib.ig_last_error().decode()
    if rc == _ffi.IG_NOT_CONVERGED:
        raise NotConverged(msg, rep, x)
    if rc == _ffi.IG_BREAKDOWN:
        raise Breakdown(msg, rep)
    _check(lib, rc, "pcg")


def richardson(a, b, precond: MgHierarchy, tol: float = 1e-10, maxit: int = 1000):
    """Preconditioned Richardson x <- x + M^{-1}(b - A x) from x = 0
    (solvers.cpp:73-120) on the device, M = one V-cycle.  Returns
    (x, ConvergenceReport); raises Diverged / NotConverged like the reference."""
    if not isinstance(precond, MgHierarchy):
        raise TypeError("richardson: the preconditioner must be a device MgHierarchy (no CPU fallback)")
    fineA = precond.A
    n = fineA.rows()
    _check_operator(a, precond, "richardson")
    if np.shape(b) != (n,):
        raise ValueError("richardson: dimension mismatch")
    bb = _as_f64(b, n)
    x = np.zeros(n)
    res = np.zeros(max(maxit, 0) + 1)
    it = C.c_int32()
    sec = C.c_double()
    lib = _ffi.gpu()
    rc = lib.ig_richardson(precond.handle, bb.ctypes.data_as(_dp), float(tol), int(maxit), x.ctypes.data_as(_dp),
                           res.ctypes.data_as(_dp), C.byref(it), C.byref(sec))
    k = it.value
    rep = ConvergenceReport(residuals=res[: k + 1].tolist(), iterations=k, converged=(rc == _ffi.IG_OK),
                            seconds=sec.value)
    if rc == _ffi.IG_OK:
        return x, rep
    msg = lib.ig_last_error().decode()
    if rc == _ffi.IG_NOT_CONVERGED:
        raise NotConverged(msg, rep, x)
    if rc == _ffi.IG_DIVERGED:
        raise Diverged(msg, rep)
    _check(lib, rc, "richardson")
