"""Per-iteration cost of the device PCG loop on C4: slope of solve time vs
maxit (tol = 0 forces NotConverged), graph vs host loop, next to the cost of
its parts (V-cycle, finest SpMV) timed alone."""
import ctypes as C
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch

    from paper_1903_10977_b200 import MgHierarchy, _ffi, build_case, configs
    lib = _ffi.gpu()
    case = build_case(configs.c4())
    h = MgHierarchy(case)
    vp = C.c_void_p
    db = torch.from_numpy(case.b).cuda()
    dx = torch.empty_like(db)
    st = torch.cuda.ExternalStream(lib.ig_hier_stream(h.handle))
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)

    def timeit(fn, n):
        fn()
        torch.cuda.synchronize()
        e0.record(st)
        for _ in range(n):
            fn()
        e1.record(st)
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / n

    for graph in (1, 0):
        lib.ig_set_option(_ffi.IG_OPT_USE_GRAPH, graph)
        t = {}
        for m in (10, 40):
            t[m] = timeit(lambda: (lib.ig_pcg_device(h.handle, vp(db.data_ptr()), 0.0, m, vp(dx.data_ptr())),
                                   lib.ig_pcg_result(h.handle, None, None)), 3)
        print(f"graph={graph}: per-iteration {(t[40] - t[10]) / 30 * 1e3:8.1f} us   (maxit 10: {t[10]:.2f} ms, 40: {t[40]:.2f} ms)")
    lib.ig_set_option(_ffi.IG_OPT_USE_GRAPH, 1)
    L = h.levels()
    tv = timeit(lambda: lib.ig_vcycle_device(h.handle, vp(db.data_ptr()), vp(dx.data_ptr())), 20)
    ts = timeit(lambda: lib.ig_level_spmv_device(h.handle, L - 1, vp(db.data_ptr()), vp(dx.data_ptr()), 0), 20)
    print(f"parts: vcycle {tv * 1e3:.1f} us, finest spmv {ts * 1e3:.1f} us, sum {(tv + ts) * 1e3:.1f} us")


if __name__ == "__main__":
    main()
