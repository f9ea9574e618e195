"""Per-level cost of the V-cycle as it really runs (CUDA graph, PDL overlap,
warm L2): time vcycle_at(l) for every level l (graph-replayed, CUDA events,
N back-to-back), so level l's marginal cost is T(l) - T(l-1) (T(0) = the
coarse solve alone).  Also the PCG iteration as a whole and the finest A p.

    python profiles/level_costs.py [c4|c3|c2|c5|c1] [--reps 200] [--json out]
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("workload", nargs="?", default="c4")
    ap.add_argument("--reps", type=int, default=200)
    ap.add_argument("--json", default=None)
    ap.add_argument("--opt", action="append", default=[], help="NAME=VALUE (ig_set_option before the hierarchy)")
    ap.add_argument("--smoother", default="as", choices=["as", "ms"])
    args = ap.parse_args()
    import numpy as np
    import torch

    import bench
    from paper_1903_10977_b200 import MgHierarchy, _ffi
    lib = _ffi.gpu()
    case, desc, _ = bench.build_workload(args.workload, 0, args.smoother)
    for kv in args.opt:
        k, v = kv.split("=")
        assert lib.ig_set_option(getattr(_ffi, "IG_OPT_" + k), int(v)) == 0, kv
    h = MgHierarchy(case)
    stream = torch.cuda.ExternalStream(lib.ig_hier_stream(h.handle))
    vp = C.c_void_p
    L = h.levels()
    out = {"workload": desc, "levels": [], "reps": args.reps}
    prev = 0.0
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for l in range(L):
        n = h._n[l]
        r = torch.from_numpy(np.random.default_rng(l).uniform(-1, 1, n)).cuda()
        x = torch.empty_like(r)
        torch.cuda.synchronize()
        for _ in range(5):
            assert lib.ig_vcycle_at_device(h.handle, l, vp(r.data_ptr()), vp(x.data_ptr())) == 0
        torch.cuda.synchronize()
        e0.record(stream)
        for _ in range(args.reps):
            lib.ig_vcycle_at_device(h.handle, l, vp(r.data_ptr()), vp(x.data_ptr()))
        e1.record(stream)
        torch.cuda.synchronize()
        t = e0.elapsed_time(e1) / args.reps * 1e3
        out["levels"].append({"level": l, "n": n, "vcycle_at_us": t, "marginal_us": t - prev})
        print(f"level {l} n={n:>9}: vcycle_at {t:8.1f} us  (+{t - prev:7.1f} us)", flush=True)
        prev = t
    # finest A p
    x = torch.from_numpy(np.ones(h._n[-1])).cuda()
    y = torch.empty_like(x)
    torch.cuda.synchronize()
    for _ in range(3):
        lib.ig_level_spmv_device(h.handle, L - 1, vp(x.data_ptr()), vp(y.data_ptr()), 0)
    torch.cuda.synchronize()
    e0.record(stream)
    for _ in range(args.reps):
        lib.ig_level_spmv_device(h.handle, L - 1, vp(x.data_ptr()), vp(y.data_ptr()), 0)
    e1.record(stream)
    torch.cuda.synchronize()
    out["finest_Ap_us"] = e0.elapsed_time(e1) / args.reps * 1e3
    # whole solve
    db = torch.from_numpy(case.b).cuda()
    dx = torch.empty_like(db)
    for _ in range(3):
        lib.ig_pcg_device(h.handle, vp(db.data_ptr()), 1e-8, 1000, vp(dx.data_ptr()))
    it = C.c_int32()
    lib.ig_pcg_result(h.handle, None, C.byref(it))
    torch.cuda.synchronize()
    e0.record(stream)
    for _ in range(5):
        lib.ig_pcg_device(h.handle, vp(db.data_ptr()), 1e-8, 1000, vp(dx.data_ptr()))
    e1.record(stream)
    torch.cuda.synchronize()
    solve_ms = e0.elapsed_time(e1) / 5
    out["solve_ms"] = solve_ms
    out["iterations"] = it.value
    vc = out["levels"][-1]["vcycle_at_us"]
    out["per_iteration_us"] = solve_ms * 1e3 / (it.value + 1)
    out["outside_vcycle_per_iteration_us"] = out["per_iteration_us"] - vc
    print(f"finest A p {out['finest_Ap_us']:.1f} us; solve {solve_ms:.2f} ms, {it.value} iterations, "
          f"{out['per_iteration_us']:.1f} us per iteration, of which V-cycle {vc:.1f} us, "
          f"outside {out['outside_vcycle_per_iteration_us']:.1f} us")
    if args.json:
        with open(args.json, "w") as f:
            json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
