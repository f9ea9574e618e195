#!/usr/bin/env python
"""Benchmark: PCG + multigrid V-cycle (additive Schwarz) solve phase on B200.

One step = one full PCG solve (zero initial guess, tol 1e-8) of the workload's
fine system, preconditioned by one V-cycle per iteration, with the host-built
hierarchy and right-hand side already resident in HBM.  `value` is
DOF-solves/s = n_dofs * n_gpus / t_step (replicas: every rank solves its own
copy, no data-path collective -- DESIGN.md "replicas only").  `e2e` is the same
metric through the C-ABI call with host buffers (ig_pcg: H2D of b, solve, D2H
of x and the residual history inside the timed region).

--impl reference times the CPU oracle (oracle/liboracle.so, the C restatement
of the reference's solve -- the reference itself cannot be built here,
SURVEY.md §0.2) on all host threads: every timed step is one COMPLETE solve
of the same workload (same hierarchy, tol, zero guess), no extrapolation.
The oracle's OpenMP loops are bit-identical to its sequential order
(oracle/oracle.c header), so the threaded run computes exactly the
single-threaded restatement.
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "PCG DOF-solves/s & V-cycle GB/s vs HBM peak (FP64); iters to 1e-8"
UNIT = "DOF-solves/s"


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md)"


class Clocks:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md clocks line)."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "20"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
        return self

    def __exit__(self, *exc):
        self.rows = []
        if self.proc is None:
            return
        self.proc.terminate()
        try:
            out, _ = self.proc.communicate(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
            out, _ = self.proc.communicate()
        for line in out.splitlines():
            parts = [x.strip() for x in line.split(",")]
            if len(parts) >= 9:
                self.rows.append(parts)

    def summary(self):
        if not getattr(self, "rows", None):
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if r[5 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


def build_workload(name: str, threads: int, smoother: str = "as"):
    from paper_1903_10977_b200 import SmootherConfig, build_case, configs
    if name == "c4":
        cfg = configs.c4(threads=threads)
        desc = ("C4: 3D [0,1]^3 128^3 minus sphere r=0.3 (seed-1 offset), p=2 B-splines, 6 levels, "
                "additive Schwarz gamma=1/27, penalty Dirichlet beta=2/h on the sphere, f=1")
    elif name == "c1":
        cfg = configs.c1(threads=threads)
        desc = "C1: 2D disc r=0.4 on 32^2, p=2 B-splines, 4 levels, additive Schwarz"
    elif name == "c3":
        cfg = configs.c3(threads=threads)
        desc = "C3: 2D plate minus 64 holes, 1024^2, p=2, 9 levels, additive Schwarz"
    elif name == "c5":
        cfg = configs.c5(threads=threads)
        desc = ("C5: 2D THB p=2, base 128^2 + 2 local refinement passes within 0.05 of the circle r=0.4, "
                "6 levels, additive Schwarz")
    elif name.startswith("c2"):
        p = int(name[3:]) if len(name) > 3 else 2
        cfg = configs.c2(p=p, seed=configs.c2_seed(), threads=threads)
        desc = f"C2: 2D disc r=0.4 on 512^2, p={p}, 8 levels, additive Schwarz, seed with eta<1e-4"
    else:
        raise SystemExit(f"unknown workload {name}")
    if smoother == "ms":  # the reference's default smoother (smoothers.hpp:17), SURVEY.md 8(f) row 1
        cfg.smoother = SmootherConfig("multiplicative-schwarz")
        desc = desc.replace("additive Schwarz gamma=1/27", "multiplicative (colored) Schwarz")
        desc = desc.replace("additive Schwarz", "multiplicative (colored) Schwarz")
    t0 = time.perf_counter()
    case = build_case(cfg)
    return case, desc, time.perf_counter() - t0


def host_cpu():
    model = "unknown"
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    return {"nproc": os.cpu_count(), "model": model}


def host_threads() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except (AttributeError, OSError):
        return os.cpu_count() or 1


def oracle_solve(case, maxit: int = 1000, threads: int = 0):
    """One oracle PCG solve (sequential-order reductions, the natural reading
    of the reference) on `threads` host threads (0 = all)."""
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import oracle_ffi as orc
    orc.set_threads(threads or host_threads())
    st, x, res, it, sec = orc.pcg(case.levels_c(), case.b, tol=1e-8, maxit=maxit, mode=orc.SEQ)
    return st, it, sec, orc.get_threads()


def common_config(desc, case, world):
    """The workload description both arms print (identical dicts)."""
    return {"workload": desc, "n_dofs": int(case.n), "nnz_finest": int(case.A.nnz),
            "levels": int(case.n_levels), "level_dofs": [int(v) for v in case.level_dofs()],
            "tol": 1e-8, "maxit": 1000, "initial_guess": "zero", "parallelism": f"replicas x{world}",
            "l2": "no flush: working set (matrix hierarchy ~3.6 GB for C4) >> 126 MB L2"}


def profile_evidence(workload: str):
    """Per-launch DRAM bytes and the binding unit of the dominant kernel, from
    the committed ncu --set full summary (profiles/spmv_traffic.json)."""
    tp = os.path.join(ROOT, "profiles", "spmv_traffic.json")
    if os.path.exists(tp):
        with open(tp) as f:
            return json.load(f).get(workload, {})
    return {}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="c4")
    ap.add_argument("--threads", type=int, default=0, help="host setup threads (0 = all)")
    ap.add_argument("--smoother", default="as", choices=["as", "ms"],
                    help="as: additive Schwarz (the BASELINE configs); ms: multiplicative colored Schwarz")
    ap.add_argument("--ref-kind", default="port", choices=["port", "reference"],
                    help="--impl reference: 'port' = the threaded oracle restatement (default: the faster, "
                         "harder CPU arm; complete solves in seconds); 'reference' = the reference's own "
                         "single-threaded solvers.cpp/multigrid.cpp/smoothers.cpp from oracle/_ref "
                         "(C4: ~3 min per complete solve, use --steps 1 --warmup 0)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-device-setup", action="store_true", help="skip the ig_hier_build setup measurement")
    ap.add_argument("--no-fast-mode", action="store_true", help="skip the tolerance-mode (fast coarse) measurement")
    ap.add_argument("--no-graph", action="store_true",
                    help="launch kernels directly instead of the CUDA graph (ncu cannot profile "
                         "kernel nodes of graphs with conditional nodes)")
    args = ap.parse_args()

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))

    if args.impl == "reference":
        return run_reference(args, world, rank)

    import numpy as np
    import torch

    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    from paper_1903_10977_b200 import MgHierarchy, _ffi
    lib = _ffi.gpu()
    if args.no_graph:
        lib.ig_set_option(_ffi.IG_OPT_USE_GRAPH, 0)

    # Host setup threads: all cores for one rank; an equal share per rank when
    # several ranks (one per GPU) build their replicas at once.
    threads = args.threads or (max(1, (os.cpu_count() or 1) // world) if world > 1 else 0)
    case, desc, t_setup = build_workload(args.workload, threads, args.smoother)
    t0 = time.perf_counter()
    h = MgHierarchy(case)
    t_upload = time.perf_counter() - t0
    info = h.info
    n = case.n
    L = info.n_levels
    log(f"[rank {rank}] {desc}: n={n} nnz={case.A.nnz} levels={L} setup={t_setup:.1f}s upload={t_upload:.1f}s")

    stream = torch.cuda.ExternalStream(lib.ig_hier_stream(h.handle))
    db = torch.from_numpy(case.b).cuda()
    dx = torch.empty_like(db)
    torch.cuda.synchronize()
    res = np.zeros(1001)
    it = C.c_int32()
    vp = C.c_void_p

    def solve():
        rc = lib.ig_pcg_device(h.handle, vp(db.data_ptr()), 1e-8, 1000, vp(dx.data_ptr()))
        assert rc == 0, lib.ig_last_error()

    def result():
        st = lib.ig_pcg_result(h.handle, res.ctypes.data_as(C.POINTER(C.c_double)), C.byref(it))
        return st, it.value

    # The clock sampler runs from the warm-up through the timed region (short
    # workloads finish the timed region faster than nvidia-smi can sample).
    clk = Clocks(local)
    clk.__enter__()
    for _ in range(max(args.warmup, 3) if args.warmup > 0 else 0):
        solve()
    st, iters = result() if args.warmup > 0 else (None, None)

    # --- timed region: K full solves, device events on the library stream ----
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    ev0.record(stream)
    for _ in range(args.steps):
        solve()
    ev1.record(stream)
    torch.cuda.synchronize()
    clk.__exit__(None, None, None)
    ms = ev0.elapsed_time(ev1) / args.steps
    st, iters = result()
    assert st == 0, f"solve did not converge (status {st})"
    if dist:
        t = torch.tensor([ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    value = n * world / (ms * 1e-3)

    # --- dominant kernel: finest-level SpMV, timed in isolation --------------
    nspmv = 20
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    py = torch.empty_like(db)
    lib.ig_level_spmv_device(h.handle, L - 1, vp(db.data_ptr()), vp(py.data_ptr()), 0)
    torch.cuda.synchronize()
    e0.record(stream)
    for _ in range(nspmv):
        lib.ig_level_spmv_device(h.handle, L - 1, vp(db.data_ptr()), vp(py.data_ptr()), 0)
    e1.record(stream)
    torch.cuda.synchronize()
    spmv_ms = e0.elapsed_time(e1) / nspmv
    hbm, peak_src = peaks()
    kernel_name = ("k_pspmv (finest A p, pattern SELL; spmv_psell.cuh)" if n > 40000
                   else "k_spmv_grp (finest A p, row-dictionary SELL)")

    # --- V-cycles/s and V-cycle GB/s (graph-replayed V-cycle) -----------------
    dz = torch.empty_like(db)
    for _ in range(3):
        lib.ig_vcycle_device(h.handle, vp(db.data_ptr()), vp(dz.data_ptr()))
    torch.cuda.synchronize()
    nv = 100  # >= 100 back-to-back V-cycles
    e0.record(stream)
    for _ in range(nv):
        lib.ig_vcycle_device(h.handle, vp(db.data_ptr()), vp(dz.data_ptr()))
    e1.record(stream)
    torch.cuda.synchronize()
    vc_ms = e0.elapsed_time(e1) / nv
    vc_gbs = info.bytes_vcycle / (vc_ms * 1e-3) / 1e9

    # --- e2e: the C-ABI call with pinned host buffers -------------------------
    hb = torch.from_numpy(case.b).pin_memory()
    hx = torch.empty(n, dtype=torch.float64).pin_memory()
    hres = np.zeros(1001)
    hit, hsec = C.c_int32(), C.c_double()
    dp = C.POINTER(C.c_double)
    for _ in range(2):
        lib.ig_pcg(h.handle, C.cast(hb.data_ptr(), dp), 1e-8, 1000, C.cast(hx.data_ptr(), dp),
                   hres.ctypes.data_as(dp), C.byref(hit), C.byref(hsec))
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    e0.record(stream)
    for _ in range(args.steps):
        rc = lib.ig_pcg(h.handle, C.cast(hb.data_ptr(), dp), 1e-8, 1000, C.cast(hx.data_ptr(), dp),
                        hres.ctypes.data_as(dp), C.byref(hit), C.byref(hsec))
        assert rc == 0
    e1.record(stream)
    torch.cuda.synchronize()
    e2e_ms = e0.elapsed_time(e1) / args.steps
    if dist:
        t = torch.tensor([e2e_ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_ms = float(t.item())
    assert np.array_equal(hx.numpy(), dx.cpu().numpy()), "host-buffer and device solves differ"

    # --- tolerance mode: explicit-inverse coarse solve ------
    fast = None
    if not args.no_fast_mode:
        lib.ig_set_option(_ffi.IG_OPT_FAST_COARSE, 1)
        lib.ig_set_option(_ffi.IG_OPT_FAST_BLOCKS, 1)
        try:
            hf = MgHierarchy(case)
        finally:
            lib.ig_set_option(_ffi.IG_OPT_FAST_COARSE, 0)
            lib.ig_set_option(_ffi.IG_OPT_FAST_BLOCKS, 0)
        xf = torch.empty_like(db)
        for _ in range(2):
            assert lib.ig_pcg_device(hf.handle, vp(db.data_ptr()), 1e-8, 1000, vp(xf.data_ptr())) == 0
        fst = lib.ig_pcg_result(hf.handle, None, C.byref(it))
        f_iters = it.value
        torch.cuda.synchronize()
        fs = torch.cuda.ExternalStream(lib.ig_hier_stream(hf.handle))
        e0.record(fs)
        for _ in range(args.steps):
            lib.ig_pcg_device(hf.handle, vp(db.data_ptr()), 1e-8, 1000, vp(xf.data_ptr()))
        e1.record(fs)
        torch.cuda.synchronize()
        f_ms = e0.elapsed_time(e1) / args.steps
        xs_, xf_ = dx.cpu().numpy(), xf.cpu().numpy()
        fast = {"what": ("tolerance mode: coarse solve and additive-Schwarz block solves as explicit-inverse "
                         "matvecs (IG_OPT_FAST_COARSE, IG_OPT_FAST_BLOCKS), not bit-identical; held to the "
                         "north-star tolerances vs the sequential oracle (tests/test_gpu_fast_mode.py)"),
                "value": n * world / (f_ms * 1e-3), "ms_per_step": f_ms, "status": int(fst),
                "iterations": f_iters,
                "x_rel_l2_vs_strict": float(np.linalg.norm(xf_ - xs_) / np.linalg.norm(xs_))}
        hf.close()

    # --- device-side hierarchy setup: ig_hier_build --
    dsetup = None
    if not args.no_device_setup:
        hd = MgHierarchy.build_on_device(case)
        wall, kern, create = hd.setup_seconds
        xd = torch.empty_like(db)
        rc = lib.ig_pcg_device(hd.handle, vp(db.data_ptr()), 1e-8, 1000, vp(xd.data_ptr()))
        assert rc == 0 and lib.ig_pcg_result(hd.handle, None, None) == 0
        same = bool(torch.equal(xd, dx))
        hd.close()
        assert same, "device-built hierarchy solves differently from the host-built one"
        dsetup = {"wall_s": wall, "device_kernels_s": kern, "hier_create_s": create,
                  "host_mg_setup_s": case.info.seconds_mg_setup,
                  "what": ("Galerkin chain + Schwarz block eigen-filter/LLT + coarsest pstrf on the device "
                           "(ig_hier_build), vs the host's multithreaded Galerkin/factorisation/pstrf "
                           "(host_mg_setup_s); hier_create_s = layout construction + upload in both paths"),
                  "solve_bit_identical": same}

    kv = info.kernels_vcycle
    launches_per_solve = (kv + 2) + iters * info.kernels_pcg_iter  # init + V-cycle + p; per iteration

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cst, cit, csec, cth = oracle_solve(case)
        assert cst == 0, f"oracle solve did not converge (status {cst})"
        cpu = {"value": n / csec, "unit": UNIT, "cores": cth, "kind": "port",
               "sample": (f"one complete {args.workload.upper()} solve ({cit} PCG iterations to 1e-8, zero "
                          f"guess, {csec:.2f} s) of oracle/liboracle.so -- the C restatement of "
                          f"solvers.cpp/multigrid.cpp/smoothers.cpp, -O3 -ffp-contract=off, sequential-order "
                          f"dots -- on {cth} host threads (OpenMP loops bit-identical to one thread)"),
               "iterations": cit, "seconds": csec, "complete_solves": 1, "host": host_cpu()}

    ev = profile_evidence(args.workload)
    traffic = ev.get("bytes_per_launch")
    layout_bytes = int(info.bytes_spmv_finest_layout)
    layout_gbs = layout_bytes / (spmv_ms * 1e-3) / 1e9
    csr_gbs = info.bytes_spmv_finest / (spmv_ms * 1e-3) / 1e9

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64",
            "data": "synthetic: seeded immersed geometry, host-assembled operator (penalty Dirichlet), f=1",
            "config": common_config(desc, case, world),
            "iterations": iters,
            "vcycles_per_s": 1e3 / vc_ms, "vcycle_ms": vc_ms, "vcycle_gbs": vc_gbs,
            "vcycle_frac_of_hbm": vc_gbs / hbm,
            "roofline": {"bound": "hbm", "kernel": kernel_name, "achieved": layout_gbs,
                         "peak": hbm, "peak_source": peak_src, "unit": "GB/s", "frac": layout_gbs / hbm,
                         "traffic": traffic, "algorithmic_bytes_per_launch": layout_bytes,
                         "launch_ms": spmv_ms,
                         "algorithmic_bytes_def": ("bytes the pattern-SELL layout must read once per launch "
                                                   "(slice metadata, deduplicated value/offset sequences, "
                                                   "per-slice and GENERAL tables, the edge gather list and "
                                                   "copy) + x, y once; launch_ms = the product as launched "
                                                   "(k_xgather + k_pspmv): DESIGN.md §5"),
                         "traffic_frac": (traffic / (spmv_ms * 1e-3) / 1e9 / hbm) if traffic else None,
                         "binding_unit": ev.get("binding_unit"),
                         "csr_equivalent": {"bytes_per_launch": int(info.bytes_spmv_finest), "gbs": csr_gbs,
                                            "frac": csr_gbs / hbm,
                                            "note": ("CSR-minimal bytes (12 B/nnz + vectors, SURVEY.md App. C) "
                                                     "that a CSR kernel would have to move for the same "
                                                     "product: an effective bandwidth, not a roofline "
                                                     "fraction")}},
            "vcycle_layout_gbs": info.bytes_vcycle_layout / (vc_ms * 1e-3) / 1e9,
            "cpu_baseline": cpu,
            "e2e": {"value": n * world / (e2e_ms * 1e-3), "unit": UNIT, "h2d_bytes_per_step": 8 * n,
                    "d2h_bytes_per_step": 8 * n + 8 * (iters + 1), "ms_per_step": e2e_ms},
            "gpu_launches": launches_per_solve * args.steps,
            "clocks": clk.summary(),
            "setup_seconds": {"host_setup": t_setup, "upload": t_upload, "device_setup": dsetup},
            "tolerance_mode": fast,
        }
        print(json.dumps(line), flush=True)
    if dist:
        dist.barrier()
        dist.destroy_process_group()


def run_reference(args, world, rank):
    """The reference arm: the oracle port (the reference cannot be built here,
    DESIGN.md §2) on all host threads.  Warm-up steps are bounded samples (the
    first 3 PCG iterations: page-in and caches, there is nothing to compile);
    every TIMED step is one complete solve."""
    if rank != 0:
        return
    case, desc, t_setup = build_workload(args.workload, args.threads, args.smoother)
    kind, what = "port", ("oracle/liboracle.so, the C restatement of the reference's solve "
                          "(sequential-order dots)")
    solve = oracle_solve
    if args.ref_kind == "reference":
        # The reference's own sources (oracle/_ref, built where /root/reference
        # exists), single-threaded like the reference.
        sys.path.insert(0, os.path.join(ROOT, "tests"))
        import reference_ffi as ref
        if not ref.available():
            print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/libimmergrid_ref.so not built"}))
            return
        rh = ref.RefHierarchy(case.levels_c())
        kind, what = "reference", ("oracle/_ref/libimmergrid_ref.so: the reference's own solvers.cpp / multigrid.cpp "
                                   "/ smoothers.cpp compiled against the Eigen stand-in (single-threaded)")

        def solve(case, maxit=1000):
            t0 = time.perf_counter()
            st, _, _, it = rh.pcg(case.b, tol=1e-8, maxit=maxit)
            return (0 if maxit < 1000 else st), it, time.perf_counter() - t0, 1
    for _ in range(args.warmup):
        solve(case, maxit=3)
    secs, its = [], []
    for _ in range(args.steps):
        st, it, sec, th = solve(case)
        assert st == 0, f"CPU solve did not converge (status {st})"
        secs.append(sec)
        its.append(it)
    t = sum(secs) / len(secs)
    v = case.n / t
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": t * 1e3, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic: seeded immersed geometry, host-assembled operator (penalty Dirichlet), f=1",
            "config": common_config(desc, case, world),
            "iterations": its[0], "complete_solves_timed": len(secs),
            "solve_seconds": {"min": min(secs), "median": statistics.median(secs), "max": max(secs)},
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": th, "kind": kind,
                             "sample": (f"{len(secs)} complete solves ({its[0]} PCG iterations each) of "
                                        f"{what}, on {th} host threads; warm-up steps = "
                                        f"the first 3 iterations")},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "setup_seconds": {"host_setup": t_setup}}
    print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
