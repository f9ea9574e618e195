"""Per-phase timing of the persistent small-level kernel (vtail.cuh) via the
%globaltimer stamps of ig_debug_tail_profile (CTA 0 after every barrier).

  IG_TAIL_ROWS=6000 IG_TAIL_CLUSTER=1 python profiles/tail_profile.py [workload]     (c5 default)
"""
import ctypes as C
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch

    from paper_1903_10977_b200 import MgHierarchy, _ffi, build_case, configs
    wl = sys.argv[1] if len(sys.argv) > 1 else "c5"
    sign = -1 if "--spmv-only" in sys.argv else 1
    mk = {"c1": configs.c1, "c2": lambda: configs.c2(2, configs.c2_seed()), "c3": configs.c3, "c4": configs.c4,
          "c5": configs.c5}
    lib = _ffi.gpu()
    lib.ig_debug_tail_profile.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.POINTER(C.c_uint64), C.c_int32,
                                          C.POINTER(C.c_int32)]
    case = build_case(mk[wl]())
    rows = int(os.environ.get("IG_TAIL_ROWS", "6000"))
    lib.ig_set_option(_ffi.IG_OPT_TAIL_ROWS, rows)
    lib.ig_set_option(_ffi.IG_OPT_TAIL_CLUSTER, int(os.environ.get("IG_TAIL_CLUSTER", "1")))
    h = MgHierarchy(case)
    r = torch.from_numpy(case.b).cuda()
    x = torch.empty_like(r)
    st = (C.c_uint64 * (257 + 64 * 1024))()
    cnt = C.c_int32()
    best = None
    for _ in range(5):
        rc = lib.ig_debug_tail_profile(h.handle, C.c_void_p(r.data_ptr()), C.c_void_p(x.data_ptr()), st,
                                       sign * (257 + 64 * 1024), C.byref(cnt))
        assert rc == 0, lib.ig_last_error()
        d = [(st[i + 1] - st[i]) / 1e3 for i in range(cnt.value - 1)]
        best = d if best is None else [min(a, b) for a, b in zip(best, d)]
    print(f"{wl}: tail kernel phases (us, min of 5): total {sum(best):.1f}")
    print("  " + " ".join(f"{v:.1f}" for v in best))
    g = st[256]
    print(f"  grid {g}: per barrier: [first arrival, last arrival (cta)] relative to the previous barrier release (us)")
    for k in range(1, cnt.value):
        arr = [st[257 + k * g + b] for b in range(g)]
        t0 = st[k - 1]
        first, last = min(arr), max(arr)
        print(f"   phase {k}: arrivals {(first - t0) / 1e3:7.1f} .. {(last - t0) / 1e3:7.1f} us (last: cta {arr.index(last)})"
              f"  barrier release +{(st[k] - last) / 1e3:.1f} us")


if __name__ == "__main__":
    main()
