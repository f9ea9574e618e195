"""ctypes declarations of the two C-ABIs (include/ig_gpu.h, include/ig_host.h).

Plain structs and function prototypes only; the reference-shaped API lives in
``paper_1903_10977_b200/__init__.py``.  Libraries are loaded from this package
directory (built in-tree by ``make -C paper_1903_10977_b200``); a missing GPU
library raises instead of falling back to anything.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))

i32, i64, f64 = C.c_int32, C.c_int64, C.c_double
P = C.POINTER


class ig_csr(C.Structure):
    _fields_ = [("n_rows", i32), ("n_cols", i32), ("nnz", i64),
                ("row_ptr", P(i32)), ("col_idx", P(i32)), ("val", P(f64))]


class ig_blocks(C.Structure):
    _fields_ = [("n_blocks", i32), ("blk_ptr", P(i32)), ("blk_dofs", P(i32)),
                ("fac_ptr", P(i64)), ("fac", P(f64)), ("n_colors", i32), ("color_of", P(i32))]


class ig_level(C.Structure):
    _fields_ = [("A", ig_csr), ("R", ig_csr), ("smoother_kind", i32),
                ("gamma", f64), ("blocks", ig_blocks)]


class ig_assembly(C.Structure):
    _fields_ = [("dim", i32), ("p", i32), ("family", i32), ("n", i32), ("n_elements", i32), ("n_tables", i32),
                ("nf", i32 * 3), ("el_ix", P(i32)), ("el_iy", P(i32)), ("el_iz", P(i32)), ("el_table", P(i32)),
                ("K", P(f64)), ("F", P(f64)), ("anchors", P(i64)), ("supp_ptr", P(i64)), ("supp_el", P(i32)),
                ("kept", P(i32))]


class ig_coarse(C.Structure):
    _fields_ = [("n", i32), ("rank", i32), ("L", P(f64)), ("piv", P(i32))]


class ig_info(C.Structure):
    _fields_ = [("n_levels", i32), ("n", i32 * 16), ("nnz_A", i64 * 16),
                ("nnz_R", i64 * 16), ("n_blocks", i32 * 16),
                ("n_multi_blocks", i32 * 16), ("sum_s", i64 * 16),
                ("sum_s2", i64 * 16), ("sell_slots_A", i64 * 16),
                ("bytes_vcycle", i64), ("bytes_pcg_iter", i64),
                ("bytes_spmv_finest", i64), ("device_bytes", i64),
                ("kernels_vcycle", i32), ("kernels_pcg_iter", i32),
                ("explicit_vals_A", i64 * 16), ("explicit_cols_A", i64 * 16),
                ("bytes_spmv_finest_layout", i64), ("bytes_vcycle_layout", i64),
                ("coarse_n", i32), ("coarse_rank", i32)]


class ig_cut3(C.Structure):
    _fields_ = [("p", i32), ("n_cut", i32), ("lo", P(f64)), ("cls", P(i32)), ("n_cls", i32 * 3),
                ("ext", P(f64) * 3), ("h", f64 * 3), ("beta", f64), ("f", f64), ("depth", i32),
                ("classify_depth", i32), ("edge_tol", f64), ("prog_len", i32), ("prog", P(f64)),
                ("gauss_tet", P(f64)), ("gauss_tri", P(f64)), ("gauss_box", P(f64)), ("table", P(i32))]


class ig_cut2(C.Structure):
    _fields_ = [("p", i32), ("n_elem", i32), ("lo", P(f64)), ("hi", P(f64)), ("cls", P(i32)), ("cut", P(i32)),
                ("sides", P(i32)), ("n_cls", i32 * 2), ("ext", P(f64) * 2), ("beta", f64), ("f", f64),
                ("depth", i32), ("classify_depth", i32), ("gauss_order", i32), ("edge_tol", f64),
                ("prog_len", i32), ("prog", P(f64)), ("gauss_q", P(f64)), ("gauss_q1", P(f64)), ("table", P(i32))]


class ig_thb_asm(C.Structure):
    _fields_ = [("p", i32), ("n", i32), ("n_elem", i32), ("lo", P(f64)), ("hi", P(f64)), ("cut", P(i32)),
                ("sides", P(i32)), ("erow_ptr", P(i32)), ("anchors", P(i32)), ("E", P(f64)),
                ("supp_ptr", P(i64)), ("supp_el", P(i32)), ("supp_li", P(i32)), ("beta", f64), ("f", f64),
                ("depth", i32), ("classify_depth", i32), ("gauss_order", i32), ("edge_tol", f64),
                ("prog_len", i32), ("prog", P(f64)), ("gauss_q", P(f64)), ("gauss_q1", P(f64))]


class igh_config(C.Structure):
    _fields_ = [("dim", i32), ("geometry", C.c_char_p), ("origin", f64 * 3),
                ("extent", f64 * 3), ("resolution", i32 * 3), ("family", i32),
                ("degree", i32), ("levels", i32), ("quad_depth", i32),
                ("gauss_order", i32), ("classify_depth", i32), ("edge_tol", f64),
                ("body_force", f64), ("beta", f64), ("dirichlet_box_sides", i32),
                ("smoother_kind", i32), ("gamma", f64), ("filter_ratio", f64),
                ("threads", i32), ("n_refine_boxes", i32), ("refine_boxes", P(f64)),
                ("refine_passes", i32), ("refine_circle", f64 * 3), ("refine_dist", f64)]


class igh_info(C.Structure):
    _fields_ = [("n_levels", i32), ("n", i32 * 16), ("nnz", i64 * 16),
                ("max_nk", i32 * 16), ("filtered_dofs", i64 * 16),
                ("coarse_rank", i32), ("cut_elements", i64), ("eta", f64),
                ("seconds_assemble", f64), ("seconds_mg_setup", f64)]


IG_OK, IG_NOT_CONVERGED, IG_BREAKDOWN, IG_INVALID_ARGUMENT, IG_CUDA_ERROR, IG_UNSUPPORTED, IG_DIVERGED = range(7)
IG_SMOOTHER_JACOBI, IG_SMOOTHER_GAUSS_SEIDEL, IG_SMOOTHER_ADDITIVE_SCHWARZ, IG_SMOOTHER_MULTIPLICATIVE_SCHWARZ = range(4)
IG_OP_A = 0
IG_OP_VCYCLE = 1
IG_OP_SMOOTHER_SYMMETRIC = 2
IG_OPT_USE_GRAPH = 1
IG_OPT_ROW_DICT = 2
IG_OPT_SMALL_ROWS = 4
IG_OPT_PSELL = 7
IG_OPT_PDL = 9
IG_OPT_RED_CTAS = 13
IG_OPT_PSELL_CTAS = 15
IG_OPT_L2_ROWS = 18
IG_OPT_L2_MB = 19
IG_OPT_COMPLEX4_ROWS = 28
IG_OPT_ONE_STREAM_ROWS = 29
IG_OPT_FAST_COARSE = 30
IG_OPT_FAST_BLOCKS = 33
IG_OPT_PSELL_PAIRS_ROWS = 32
IG_OPT_GAL_SHORT = 21
IG_OPT_PSELL_CTAB = 23
IG_OPT_PSELL_LINES2 = 27
IG_OPT_PSELL_MULTI = 34
IG_OPT_PSELL_AB = 35
IG_OPT_PSELL_ROWS4 = 36
IG_OPT_PSELL_EDGE_ROWS = 37
IG_OPT_PSELL_ROWS4_ROWS = 38
IG_OPT_PSELL_ORDER = 39

_host = None
_gpu = None


def _lib(name: str) -> C.CDLL:
    path = os.path.join(HERE, name)
    if not os.path.exists(path):
        raise RuntimeError(f"{path} is not built; run `make -C {HERE}` (or __graft_entry__.build())")
    return C.CDLL(path)


def host() -> C.CDLL:
    global _host
    if _host is None:
        lib = _lib("libig_host.so")
        lib.igh_config_default.argtypes = [P(igh_config)]
        lib.igh_config_default.restype = None
        lib.igh_build.argtypes = [P(igh_config), P(C.c_void_p)]
        lib.igh_build_geometry.argtypes = [P(igh_config), P(C.c_void_p)]
        lib.igh_levels.argtypes = [C.c_void_p, P(P(ig_level)), P(i32), P(P(ig_coarse))]
        lib.igh_rhs.argtypes = [C.c_void_p, P(i32)]
        lib.igh_rhs.restype = P(f64)
        lib.igh_assembly_payload.argtypes = [C.c_void_p, P(ig_assembly)]
        lib.igh_prefilter_blocks.argtypes = [C.c_void_p, i32, P(i32), P(P(i32)), P(P(i32))]
        lib.igh_get_info.argtypes = [C.c_void_p, P(igh_info)]
        lib.igh_support_fraction.argtypes = [C.c_void_p, P(f64)]
        lib.igh_cut3_payload.argtypes = [C.c_void_p, P(ig_cut3)]
        lib.igh_cut2_payload.argtypes = [C.c_void_p, P(ig_cut2)]
        lib.igh_thb_payload.argtypes = [C.c_void_p, P(ig_thb_asm)]
        lib.igh_anchors.argtypes = [C.c_void_p, i32, P(i32)]
        lib.igh_write.argtypes = [C.c_void_p, C.c_char_p]
        lib.igh_read.argtypes = [C.c_char_p, P(C.c_void_p)]
        lib.igh_destroy.argtypes = [C.c_void_p]
        lib.igh_destroy.restype = None
        lib.igh_last_error.restype = C.c_char_p
        lib.igh_pstrf.argtypes = [i32, P(f64), P(i32), f64]
        lib.igh_pstrf.restype = i32
        lib.igh_eta.argtypes = [P(igh_config), P(f64), P(i64), P(i32)]
        _host = lib
    return _host


GPU_SYMBOLS = (
    "ig_hier_create", "ig_hier_destroy", "ig_hier_info", "ig_hier_stream",
    "ig_vcycle", "ig_vcycle_at", "ig_coarse_solve", "ig_smoother_apply",
    "ig_level_spmv", "ig_pcg", "ig_vcycle_device", "ig_level_spmv_device", "ig_pcg_device",
    "ig_pcg_result", "ig_last_error", "ig_set_option", "ig_richardson",
    "ig_smoother_apply_dir", "ig_smoother_apply_symmetric", "ig_galerkin_hierarchy", "ig_csr_free",
    "ig_factorize_blocks", "ig_blocks_free", "ig_pstrf", "ig_hier_build",
    "ig_operator_columns", "ig_assemble", "ig_hier_set_option", "ig_hier_matches", "ig_vcycle_at_device", "ig_cut_quadrature3", "ig_cut_quadrature2", "ig_assemble_thb",
)


def gpu() -> C.CDLL:
    global _gpu
    if _gpu is None:
        lib = _lib(os.environ.get("IG_GPU_LIB", "libig_gpu.so"))  # variant builds for profiling only
        vp, dp = C.c_void_p, P(f64)
        lib.ig_hier_create.argtypes = [P(ig_level), i32, P(ig_coarse), P(vp)]
        lib.ig_galerkin_hierarchy.argtypes = [P(ig_csr), P(ig_csr), i32, P(ig_csr), dp]
        lib.ig_csr_free.argtypes = [P(ig_csr)]
        lib.ig_csr_free.restype = None
        lib.ig_factorize_blocks.argtypes = [P(ig_csr), i32, P(i32), P(i32), f64, P(ig_blocks), P(i64), dp]
        lib.ig_blocks_free.argtypes = [P(ig_blocks)]
        lib.ig_blocks_free.restype = None
        lib.ig_pstrf.argtypes = [i32, dp, P(i32), f64, P(i32)]
        lib.ig_operator_columns.argtypes = [vp, i32, i32, i32, dp]
        lib.ig_assemble.argtypes = [P(ig_assembly), P(ig_csr), dp, dp]
        lib.ig_hier_build.argtypes = [P(ig_csr), P(ig_csr), P(ig_blocks), dp, i32, f64, i32, P(vp), dp]
        lib.ig_hier_destroy.argtypes = [vp]
        lib.ig_hier_destroy.restype = None
        lib.ig_hier_info.argtypes = [vp, P(ig_info)]
        lib.ig_hier_stream.argtypes = [vp]
        lib.ig_hier_stream.restype = vp
        lib.ig_vcycle.argtypes = [vp, dp, dp]
        lib.ig_vcycle_at.argtypes = [vp, i32, dp, dp]
        lib.ig_coarse_solve.argtypes = [vp, dp, dp]
        lib.ig_smoother_apply.argtypes = [vp, i32, dp, dp]
        lib.ig_smoother_apply_dir.argtypes = [vp, i32, dp, dp, i32]
        lib.ig_smoother_apply_symmetric.argtypes = [vp, i32, dp, dp]
        lib.ig_level_spmv.argtypes = [vp, i32, dp, dp, i32]
        lib.ig_pcg.argtypes = [vp, dp, f64, i32, dp, dp, P(i32), dp]
        lib.ig_richardson.argtypes = [vp, dp, f64, i32, dp, dp, P(i32), dp]
        lib.ig_vcycle_device.argtypes = [vp, vp, vp]
        lib.ig_vcycle_at_device.argtypes = [vp, i32, vp, vp]
        lib.ig_level_spmv_device.argtypes = [vp, i32, vp, vp, i32]
        lib.ig_debug_vcycle_timeline.argtypes = [vp, vp, vp, i32, P(C.c_float), P(i32), C.c_char_p, i32, P(i32)]
        lib.ig_pcg_device.argtypes = [vp, vp, f64, i32, vp]
        lib.ig_pcg_result.argtypes = [vp, dp, P(i32)]
        lib.ig_last_error.restype = C.c_char_p
        lib.ig_set_option.argtypes = [i32, i64]
        lib.ig_hier_set_option.argtypes = [vp, i32, i64]
        lib.ig_hier_matches.argtypes = [vp, P(ig_csr)]
        lib.ig_cut_quadrature3.argtypes = [P(ig_cut3), dp, dp, dp, dp]
        lib.ig_cut_quadrature2.argtypes = [P(ig_cut2), dp, dp, dp, dp]
        lib.ig_assemble_thb.argtypes = [P(ig_thb_asm), P(ig_csr), dp, dp]
        _gpu = lib
    return _gpu
