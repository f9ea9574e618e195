"""One multiplicative-Schwarz V-cycle (direct launches) for ncu launch lists.

  python profiles/profile_ms.py [c4|c5]
"""
import ctypes as C
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch

    from paper_1903_10977_b200 import MgHierarchy, SmootherConfig, _ffi, build_case, configs
    wl = sys.argv[1] if len(sys.argv) > 1 else "c5"
    cfg = {"c4": configs.c4, "c5": configs.c5}[wl]()
    cfg.smoother = SmootherConfig("multiplicative-schwarz")
    case = build_case(cfg)
    h = MgHierarchy(case)
    lib = _ffi.gpu()
    lib.ig_set_option(_ffi.IG_OPT_USE_GRAPH, 0)
    vp = C.c_void_p
    db = torch.from_numpy(case.b).cuda()
    dx = torch.empty_like(db)
    torch.cuda.synchronize()
    assert lib.ig_vcycle_device(h.handle, vp(db.data_ptr()), vp(dx.data_ptr())) == 0
    torch.cuda.synchronize()
    print("done", case.n)


if __name__ == "__main__":
    main()
