"""Small driver for ncu captures of the C4 (3D 128^3) kernels.

  python profiles/profile_c4.py spmv     # 3 finest-level SpMVs (A p)
  python profiles/profile_c4.py vcycle   # one V-cycle, direct launches (no graph)
  python profiles/profile_c4.py vcycle2  # two V-cycles (profile the second, warm L2)
  python profiles/profile_c4.py pcg      # one solve capped at 2 iterations

Never a timing source: numbers printed under ncu are not bench values.
"""
import ctypes as C
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch

    from paper_1903_10977_b200 import MgHierarchy, _ffi, build_case, configs
    mode = sys.argv[1] if len(sys.argv) > 1 else "spmv"
    res = int(os.environ.get("IG_PROFILE_RES", "128"))
    case = build_case(configs.c4(res=res, levels=6 if res == 128 else 5))
    h = MgHierarchy(case)
    lib = _ffi.gpu()
    vp = C.c_void_p
    db = torch.from_numpy(case.b).cuda()
    dx = torch.empty_like(db)
    torch.cuda.synchronize()
    L = h.levels()
    if mode == "spmv":
        for _ in range(3):
            assert lib.ig_level_spmv_device(h.handle, L - 1, vp(db.data_ptr()), vp(dx.data_ptr()), 0) == 0
    elif mode in ("vcycle", "vcycle2"):
        lib.ig_hier_set_option(h.handle, _ffi.IG_OPT_USE_GRAPH, 0)
        for _ in range(2 if mode == "vcycle2" else 1):
            assert lib.ig_vcycle_device(h.handle, vp(db.data_ptr()), vp(dx.data_ptr())) == 0
    elif mode == "pcg":
        lib.ig_hier_set_option(h.handle, _ffi.IG_OPT_USE_GRAPH, 0)
        assert lib.ig_pcg_device(h.handle, vp(db.data_ptr()), 1e-8, 2, vp(dx.data_ptr())) == 0
        lib.ig_pcg_result(h.handle, None, None)
    torch.cuda.synchronize()
    print("profile driver done:", mode, case.n)


if __name__ == "__main__":
    main()
