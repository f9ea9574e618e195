"""Device time of one level SpMV (A x, direct launch, CUDA events over 50
launches) for every level of a workload: which layout/kernel each level gets
and what it costs.

  python profiles/level_spmv.py [workload]     (c5 default)
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
    mk = {"c1": configs.c1, "c2": lambda: configs.c2(2, configs.c2_seed()), "c3": configs.c3, "c4": configs.c4,
          "c5": configs.c5}
    lib = _ffi.gpu()
    case = build_case(mk[wl]())
    h = MgHierarchy(case)
    vp = C.c_void_p
    st = torch.cuda.ExternalStream(lib.ig_hier_stream(h.handle))
    n = case.n
    x = torch.ones(n, dtype=torch.float64, device="cuda")
    y = torch.empty_like(x)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for l in range(1, h.levels()):
        for mode in (0, 2, 3):
            f = lambda: lib.ig_level_spmv_device(h.handle, l, vp(x.data_ptr()), vp(y.data_ptr()), mode)
            for _ in range(3):
                f()
            torch.cuda.synchronize()
            e0.record(st)
            for _ in range(50):
                f()
            e1.record(st)
            torch.cuda.synchronize()
            print(f"{wl} L{l} n={h._n[l]:8d} mode {mode}: {e0.elapsed_time(e1) / 50 * 1e3:8.2f} us", flush=True)


if __name__ == "__main__":
    main()
