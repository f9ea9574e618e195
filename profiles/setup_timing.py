"""Wall-time breakdown of the device setup pipeline (setup_on_device) against
the host pipeline (build_case + MgHierarchy) for one config.

    IG_TIMING=1 python profiles/setup_timing.py [c4|c3|c2|c5] [--json out]
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("workload", nargs="?", default="c4")
    ap.add_argument("--json", default=None)
    ap.add_argument("--no-host", action="store_true")
    args = ap.parse_args()
    import numpy as np  # noqa: F401

    import paper_1903_10977_b200 as pkg
    from paper_1903_10977_b200 import MgHierarchy, build_case, configs
    cfg = {"c2": lambda: configs.c2(p=2, seed=configs.c2_seed()), "c3": configs.c3, "c4": configs.c4,
           "c5": configs.c5}[args.workload]()
    pkg._ffi.gpu()
    import torch
    torch.zeros(1).cuda()  # context up before timing
    out = {"workload": args.workload}
    t = {}
    t0 = time.perf_counter()
    geo = build_case(cfg, geometry_only=True)
    t["host_geometry"] = time.perf_counter() - t0
    thb = geo.config.family == "thb"
    if not thb:
        t0 = time.perf_counter()
        table, Kc, Fc, _, qs = pkg.cut_quadrature_on_device(geo)
        t["cut_quadrature_call"] = time.perf_counter() - t0
        t["cut_quadrature_device"] = qs
    t0 = time.perf_counter()
    A, b, asec = pkg.assemble_on_device(geo, device_cut=True)
    t["assemble_on_device_call"] = time.perf_counter() - t0
    t["ig_assemble_wall"], t["ig_assemble_device"] = asec
    t0 = time.perf_counter()
    h = MgHierarchy.build_on_device(geo, A)
    t["build_on_device_call"] = time.perf_counter() - t0
    t["ig_hier_build_wall"], t["ig_hier_build_device"], t["ig_hier_create"] = h.setup_seconds
    h.close()
    t0 = time.perf_counter()
    ds = pkg.setup_on_device(cfg)
    t["setup_on_device_total"] = time.perf_counter() - t0
    out["setup_on_device_seconds"] = ds.seconds
    ds.close()
    if not args.no_host:
        t0 = time.perf_counter()
        case = build_case(cfg)
        t["host_build_case"] = time.perf_counter() - t0
        t0 = time.perf_counter()
        hh = MgHierarchy(case)
        t["host_hier_create"] = time.perf_counter() - t0
        t["host_total"] = t["host_build_case"] + t["host_hier_create"]
        hh.close()
        case.close()
    out["seconds"] = t
    out["threads"] = os.cpu_count()
    print(json.dumps(out, indent=1))
    if args.json:
        with open(args.json, "w") as f:
            json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
