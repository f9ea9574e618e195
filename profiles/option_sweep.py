"""Sweep one ig_set_option over values on several workloads: V-cycle and full
PCG device time (CUDA events on the library stream).

  [IG_PRESET=opt=val,...] python profiles/option_sweep.py OPTION v1,v2,... [workloads]
  e.g.  python profiles/option_sweep.py 4 0,50000,300000 c4,c3,c2
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
    for kv in filter(None, os.environ.get("IG_PRESET", "").split(",")):  # e.g. IG_PRESET=19=96,18=300000
        k, v = kv.split("=")
        assert lib.ig_set_option(int(k), int(v)) == 0
    opt = int(sys.argv[1])
    vals = [int(v) for v in sys.argv[2].split(",")]
    wls = sys.argv[3].split(",") if len(sys.argv) > 3 else ["c4"]
    mk = {"c1": configs.c1, "c2": lambda: configs.c2(2, configs.c2_seed()), "c3": configs.c3, "c4": configs.c4,
          "c5": configs.c5}
    vp = C.c_void_p
    for wl in wls:
        case = build_case(mk[wl]())
        db = torch.from_numpy(case.b).cuda()
        dx = torch.empty_like(db)
        for v in vals:
            lib.ig_set_option(opt, v)
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
            ts = timeit(lambda: lib.ig_level_spmv_device(h.handle, L - 1, vp(db.data_ptr()), vp(dx.data_ptr()), 0), 20)
            tv = timeit(lambda: lib.ig_vcycle_device(h.handle, vp(db.data_ptr()), vp(dx.data_ptr())), 20)
            tp = timeit(lambda: lib.ig_pcg_device(h.handle, vp(db.data_ptr()), 1e-8, 1000, vp(dx.data_ptr())), 3)
            it = C.c_int32()
            lib.ig_pcg_result(h.handle, None, C.byref(it))
            print(f"{wl} option {opt}={v}: spmv {ts * 1e3:7.1f} us ({h.info.bytes_spmv_finest_layout / 1e6:.0f} MB layout)"
                  f"  vcycle {tv * 1e3:8.1f} us  pcg {tp:8.3f} ms  iters {it.value}", flush=True)
            h.close()
            torch.cuda.synchronize()


if __name__ == "__main__":
    main()
