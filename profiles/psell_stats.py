"""Slice statistics of the pattern-SELL layout (host only, no GPU):
python profiles/psell_stats.py [workload] [res]   (caches the CSR under gpurun_out/)"""
import ctypes as C
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def load(wl, res, which="A"):
    from paper_1903_10977_b200 import build_case, configs
    base = os.path.join(ROOT, "gpurun_out", f"csr_{wl}_{res}" + ("" if which == "A" else "_" + which))
    if os.path.exists(base + "_val.npy"):
        return tuple(np.load(base + s, mmap_mode="r") for s in ("_ptr.npy", "_col.npy", "_val.npy"))
    cfg = configs.c4(res=res, levels=configs.c4_levels(res)) if wl == "c4" else configs.CONFIGS[wl]()
    case = build_case(cfg)
    A = case.A.to_scipy().tocsr()
    if which.startswith("L"):  # level operator A_l, e.g. L4
        A = case.level_A(int(which[1:])).to_scipy().tocsr()
        A.sort_indices()
    if which in ("P", "R"):
        from paper_1903_10977_b200 import SpMat
        R = SpMat.from_c(case._lv[case.n_levels - 1].R, case).to_scipy().tocsr()
        A = R.T.tocsr() if which == "P" else R
        A.sort_indices()
    os.makedirs(os.path.dirname(base), exist_ok=True)
    np.save(base + "_ptr.npy", A.indptr.astype(np.int32))
    np.save(base + "_col.npy", A.indices.astype(np.int32))
    np.save(base + "_val.npy", A.data)
    return A.indptr.astype(np.int32), A.indices.astype(np.int32), A.data


def main():
    from paper_1903_10977_b200 import _ffi
    wl = sys.argv[1] if len(sys.argv) > 1 else "c4"
    res = int(sys.argv[2]) if len(sys.argv) > 2 else 128
    which = sys.argv[3] if len(sys.argv) > 3 else "A"
    ptr, col, val = (np.ascontiguousarray(a) for a in load(wl, res, which))
    lib = _ffi.gpu()
    a = _ffi.ig_csr()
    a.n_rows = len(ptr) - 1
    a.n_cols = int(col.max()) + 1 if which in ("P", "R") else a.n_rows
    a.nnz = len(col)
    a.row_ptr = ptr.ctypes.data_as(C.POINTER(C.c_int32))
    a.col_idx = col.ctypes.data_as(C.POINTER(C.c_int32))
    a.val = val.ctypes.data_as(C.POINTER(C.c_double))
    out = (C.c_int64 * 32)()
    lib.ig_debug_psell_stats.argtypes = [C.POINTER(_ffi.ig_csr), C.POINTER(C.c_int64), C.c_int32]
    rc = lib.ig_debug_psell_stats(C.byref(a), out, 32)
    assert rc == 0, rc
    o = list(out)
    names = ["GENERAL", "FAST", "FAST2", "FAST4", "FAST2M"]
    for k in range(5):
        print(f"{names[k]:8s}: {o[k]:7d} slices, {o[5 + k]:9d} lanes used, by lanes (1-8, 9-16, 17-24, 25-32): {o[10 + 4 * k:14 + 4 * k]}")
    print(f"layout bytes {o[30]}, table rows {o[31]}")
    print("total slices", sum(o[:5]))


if __name__ == "__main__":
    main()
