"""Variant sweep on C4: row-dictionary on/off x SpMV code variants.
Prints finest SpMV time, V-cycle time and full PCG solve time (CUDA events
on the library stream).  Used to choose the defaults."""
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
    vp = C.c_void_p
    db = torch.from_numpy(case.b).cuda()
    dx = torch.empty_like(db)
    variants = [int(v) for v in (sys.argv[1].split(",") if len(sys.argv) > 1 else "0,1,2,3".split(","))]
    dicts = [int(v) for v in (sys.argv[2].split(",") if len(sys.argv) > 2 else "1".split(","))]
    for dct in dicts:
        lib.ig_set_option(_ffi.IG_OPT_ROW_DICT, dct)
        for var in variants:
            lib.ig_set_option(_ffi.IG_OPT_SPMV_VARIANT, var)
            h = MgHierarchy(case)
            L = h.levels()
            st = torch.cuda.ExternalStream(lib.ig_hier_stream(h.handle))
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)

            def timeit(fn, n):
                for _ in range(2):
                    fn()
                torch.cuda.synchronize()
                e0.record(st)
                for _ in range(n):
                    fn()
                e1.record(st)
                torch.cuda.synchronize()
                return e0.elapsed_time(e1) / n

            t_spmv = timeit(lambda: lib.ig_level_spmv_device(h.handle, L - 1, vp(db.data_ptr()), vp(dx.data_ptr()), 0), 20)
            t_vc = timeit(lambda: lib.ig_vcycle_device(h.handle, vp(db.data_ptr()), vp(dx.data_ptr())), 20)
            t_pcg = timeit(lambda: lib.ig_pcg_device(h.handle, vp(db.data_ptr()), 1e-8, 1000, vp(dx.data_ptr())), 3)
            it = C.c_int32()
            lib.ig_pcg_result(h.handle, None, C.byref(it))
            info = h.info
            print(f"dict={dct} var={var}: spmv {t_spmv * 1e3:7.1f} us ({info.bytes_spmv_finest_layout / t_spmv / 1e6:6.0f} GB/s layout)"
                  f"  vcycle {t_vc * 1e3:7.1f} us  pcg {t_pcg:7.2f} ms  iters {it.value}", flush=True)
            h.close()
            torch.cuda.synchronize()


if __name__ == "__main__":
    main()
