"""Finest-level pattern-SELL products timed alone (CUDA events on the library
stream): A x, r - A x (distinct and in-place), restriction, prolongation.
  python profiles/spmv_modes.py [workload] [level]"""
import ctypes as C
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch

    from paper_1903_10977_b200 import MgHierarchy, _ffi, build_case, configs
    lib = _ffi.gpu()
    wl = sys.argv[1] if len(sys.argv) > 1 else "c4"
    mk = {"c1": configs.c1, "c2": lambda: configs.c2(2, configs.c2_seed()), "c3": configs.c3, "c4": configs.c4,
          "c5": configs.c5}
    case = build_case(mk[wl]())
    h = MgHierarchy(case)
    L = int(sys.argv[2]) + 1 if len(sys.argv) > 2 else h.info.n_levels  # optional level (default: finest)
    n, nc = h.info.n[L - 1], h.info.n[L - 2]
    vp = C.c_void_p
    g = torch.Generator(device="cuda").manual_seed(1)
    x = torch.rand(n, dtype=torch.float64, device="cuda", generator=g)
    y = torch.rand(n, dtype=torch.float64, device="cuda", generator=g)
    xc = torch.rand(nc, dtype=torch.float64, device="cuda", generator=g)
    yc = torch.empty(nc, dtype=torch.float64, device="cuda")
    st = torch.cuda.ExternalStream(lib.ig_hier_stream(h.handle))
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)

    def timeit(fn, reps=50):
        fn()
        torch.cuda.synchronize()
        e0.record(st)
        for _ in range(reps):
            fn()
        e1.record(st)
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / reps * 1e3

    sp = lib.ig_level_spmv_device
    print(f"{wl} level {L - 1} n={n}")
    print(f"  A x            {timeit(lambda: sp(h.handle, L - 1, vp(x.data_ptr()), vp(y.data_ptr()), 0)):7.1f} us")
    print(f"  r - A x        {timeit(lambda: sp(h.handle, L - 1, vp(x.data_ptr()), vp(y.data_ptr()), 1)):7.1f} us")
    print(f"  restriction    {timeit(lambda: sp(h.handle, L - 1, vp(x.data_ptr()), vp(yc.data_ptr()), 2)):7.1f} us")
    print(f"  prolongation   {timeit(lambda: sp(h.handle, L - 1, vp(xc.data_ptr()), vp(y.data_ptr()), 3)):7.1f} us")
    h.close()


if __name__ == "__main__":
    main()
