"""Warm per-step timeline of one V-cycle (CUDA events between steps, direct
launches): where the V-cycle time goes, level by level.

  python profiles/vcycle_timeline.py [workload]     (c4 default)
"""
import ctypes as C
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch

    from paper_1903_10977_b200 import MgHierarchy, _ffi, build_case, configs
    wl = sys.argv[1] if len(sys.argv) > 1 else "c4"
    mk = {"c1": configs.c1, "c2": lambda: configs.c2(2, configs.c2_seed()), "c3": configs.c3, "c4": configs.c4,
          "c5": configs.c5}
    lib = _ffi.gpu()
    case = build_case(mk[wl]())
    h = MgHierarchy(case)
    db = torch.from_numpy(case.b).cuda()
    dx = torch.empty_like(db)
    torch.cuda.synchronize()
    N, LL = 256, 24
    ms = (C.c_float * N)()
    lev = (C.c_int32 * N)()
    lab = C.create_string_buffer(N * LL)
    cnt = C.c_int32()
    best = None
    for _ in range(5):
        rc = lib.ig_debug_vcycle_timeline(h.handle, C.c_void_p(db.data_ptr()), C.c_void_p(dx.data_ptr()), N, ms, lev,
                                          lab, LL, C.byref(cnt))
        assert rc == 0, lib.ig_last_error()
        cur = [ms[i] for i in range(cnt.value)]
        best = cur if best is None else [min(a, b) for a, b in zip(best, cur)]
    tot = sum(best)
    print(f"{wl}: one V-cycle, direct launches, {tot * 1e3:.1f} us (min over 5 per step)")
    per = {}
    for i in range(cnt.value):
        name = lab.raw[i * LL:(i + 1) * LL].split(b"\0")[0].decode()
        key = (lev[i], name)
        per[key] = per.get(key, 0.0) + best[i]
        print(f"  L{lev[i]} {name:12s} {best[i] * 1e3:8.1f} us")
    by_level = {}
    for (l, _), t in per.items():
        by_level[l] = by_level.get(l, 0.0) + t
    print("  per level:", ", ".join(f"L{l}: {t * 1e3:.0f} us" for l, t in sorted(by_level.items(), reverse=True)))


if __name__ == "__main__":
    main()
