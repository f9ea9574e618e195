"""Tuning sweep of one library build (IG_GPU_LIB=libig_gpu_<variant>.so, see
profiles/build_variants.sh) over workloads x IG_OPT_PSELL_CTAS (pattern-SELL
occupancy cap).  Finest SpMV, V-cycle and PCG device time (CUDA events on
the library stream).

  python profiles/psell_sweep.py [workloads] [ctas]     e.g.  c4,c5 0,3,4
"""
import ctypes as C
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch

    from paper_1903_10977_b200 import MgHierarchy, _ffi, build_case, configs
    lib = _ffi.gpu()
    wls = (sys.argv[1] if len(sys.argv) > 1 else "c4").split(",")
    ctas = [int(v) for v in (sys.argv[2] if len(sys.argv) > 2 else "0").split(",")]
    mk = {"c1": configs.c1, "c2": lambda: configs.c2(2, configs.c2_seed()), "c3": configs.c3, "c4": configs.c4,
          "c5": configs.c5}
    vp = C.c_void_p
    tag = os.environ.get("IG_GPU_LIB", "libig_gpu.so")
    for kv in filter(None, os.environ.get("IG_OPTS", "").split(",")):  # e.g. IG_OPTS=34=0,27=1
        k, v = kv.split("=")
        assert lib.ig_set_option(int(k), int(v)) == 0
        tag += f" opt{k}={v}"
    for wl in wls:
        case = build_case(mk[wl]())
        db = torch.from_numpy(case.b).cuda()
        dx = torch.empty_like(db)
        h = MgHierarchy(case)
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

        L = h.info.n_levels
        for c in ctas:
            assert lib.ig_set_option(_ffi.IG_OPT_PSELL_CTAS, c) == 0
            ts = timeit(lambda: lib.ig_level_spmv_device(h.handle, L - 1, vp(db.data_ptr()), vp(dx.data_ptr()), 0), 20)
            tv = timeit(lambda: lib.ig_vcycle_device(h.handle, vp(db.data_ptr()), vp(dx.data_ptr())), 20)
            tp = timeit(lambda: lib.ig_pcg_device(h.handle, vp(db.data_ptr()), 1e-8, 1000, vp(dx.data_ptr())), 3)
            it = C.c_int32()
            lib.ig_pcg_result(h.handle, None, C.byref(it))
            print(f"{tag} {wl} ctas={c}: spmv {ts * 1e3:7.1f} us  vcycle {tv * 1e3:8.1f} us  "
                  f"pcg {tp:8.3f} ms  iters {it.value}", flush=True)
        h.close()
        torch.cuda.synchronize()


if __name__ == "__main__":
    main()
