"""N1 (north star): mesh- and cut-independent iteration counts on the C4
family (3D cube minus a sphere r = 0.3, p = 2 B-splines, coarsest grid 4^3),
on the device and on the CPU oracle.

Resolutions 16^3..128^3 x sphere-offset seeds 1..8, additive Schwarz (the
BASELINE configs) and multiplicative (colored) Schwarz (the reference's
default smoother).  The oracle (sequential-order dots) runs where it takes
seconds (all host threads); the device count is bit-identical to the
GPU-order oracle (tests/test_gpu_parity.py), so the oracle column pins the
reference-order count.  Writes profiles/<out>.json and prints a markdown
table.

    python profiles/n1_iterations.py --out r02_n1_iterations
"""
from __future__ import annotations

import argparse
import dataclasses
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default="r02_n1_iterations")
    ap.add_argument("--res", default="16,32,64,128")
    ap.add_argument("--seeds", default="1,2,3,4,5,6,7,8")
    ap.add_argument("--smoothers", default="as,ms")
    ap.add_argument("--oracle-max-dofs", type=int, default=300_000,
                    help="run the CPU oracle up to this many DOFs (AS); MS up to a tenth of it")
    args = ap.parse_args()

    import oracle_ffi as orc
    from paper_1903_10977_b200 import MgHierarchy, SmootherConfig, build_case, configs, pcg

    rows = []
    for sm in args.smoothers.split(","):
        for res in (int(r) for r in args.res.split(",")):
            for seed in (int(s) for s in args.seeds.split(",")):
                cfg = configs.c4(res=res, levels=configs.c4_levels(res), seed=seed)
                if sm == "ms":
                    cfg = dataclasses.replace(cfg, smoother=SmootherConfig("multiplicative-schwarz"))
                t0 = time.perf_counter()
                case = build_case(cfg)
                t_setup = time.perf_counter() - t0
                h = MgHierarchy(case)
                x, rep = pcg(h.A, case.b, h, tol=1e-8, maxit=1000)
                row = {"smoother": sm, "res": res, "seed": seed, "n": case.n, "levels": case.n_levels,
                       "eta": case.info.eta, "cut_elements": int(case.info.cut_elements),
                       "gpu_iterations": rep.iterations, "gpu_converged": rep.converged,
                       "gpu_solve_s": rep.seconds, "setup_s": t_setup, "oracle_seq_iterations": None}
                lim = args.oracle_max_dofs if sm == "as" else args.oracle_max_dofs // 10
                if case.n <= lim:
                    st, _, _, it, sec = orc.pcg(case.levels_c(), case.b, tol=1e-8, maxit=1000, mode=orc.SEQ)
                    row["oracle_seq_iterations"] = it if st == 0 else None
                    row["oracle_s"] = sec
                h.close()
                rows.append(row)
                print(json.dumps(row), flush=True)

    out = {"what": __doc__.strip().splitlines()[0], "rows": rows}
    with open(os.path.join(ROOT, "profiles", args.out + ".json"), "w") as f:
        json.dump(out, f, indent=1)

    # Markdown summary: per smoother x resolution, min / max over seeds.
    lines = ["| smoother | res | n (seed 1) | iterations over seeds (device) | min..max | oracle SEQ (seeds run) |",
             "|---|---|---|---|---|---|"]
    for sm in args.smoothers.split(","):
        for res in (int(r) for r in args.res.split(",")):
            rr = [r for r in rows if r["smoother"] == sm and r["res"] == res]
            its = [r["gpu_iterations"] for r in rr]
            orcs = [r["oracle_seq_iterations"] for r in rr if r["oracle_seq_iterations"] is not None]
            lines.append(f"| {sm} | {res}^3 | {rr[0]['n']:,} | {' '.join(map(str, its))} | {min(its)}..{max(its)} | "
                         f"{' '.join(map(str, orcs)) if orcs else '-'} |")
    md = "\n".join(lines)
    with open(os.path.join(ROOT, "profiles", args.out + ".md"), "w") as f:
        f.write(md + "\n")
    print(md)


if __name__ == "__main__":
    main()
