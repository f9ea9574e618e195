"""Per-kernel table of one V-cycle: device time and DRAM bytes from an ncu
launch list (gpu__time_duration.sum, dram__bytes_read.sum,
dram__bytes_write.sum of `profiles/profile_c4.py vcycle` or
`profiles/profile_c5.py`), next to each kernel's ALGORITHMIC bytes
(CSR-minimal) and the fraction of the measured copy
bandwidth it reaches.  Runs on the CPU (rebuilds the case to size the kernels).

  python profiles/vcycle_kernel_table.py gpurun_out/vc_c4_kernels.csv c4 > profiles/r01_vcycle_kernels_c4.md
"""
import csv
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def ncu_records(path):
    rows = list(csv.reader(open(path)))
    h, recs, order = None, {}, []
    for r in rows:
        if len(r) > 5 and r[0] == "ID":
            h = r
            continue
        if h and len(r) == len(h):
            d = dict(zip(h, r))
            k = int(d["ID"])
            if k not in recs:
                recs[k] = {"name": d["Kernel Name"].split("(")[0].replace("void ", "")}
                order.append(k)
            v = d["Metric Value"].replace(",", "")
            scale = {"ns": 1e-3, "us": 1.0, "ms": 1e3, "byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
            recs[k][d["Metric Name"]] = float(v) * scale.get(d["Metric Unit"], 1.0) if v not in ("", "n/a") else None
    return [recs[k] for k in order]


def main():
    from paper_1903_10977_b200 import build_case, configs
    path, wl = sys.argv[1], sys.argv[2]
    small = int(sys.argv[3]) if len(sys.argv) > 3 else 10000
    case = build_case({"c4": configs.c4, "c5": configs.c5, "c3": configs.c3}[wl]())
    L = case.n_levels
    peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
    lv = {}
    for l in range(1, L):
        n = case.level_dofs()[l]
        nc = case.level_dofs()[l - 1]
        ptr, dofs, _, _ = case.blocks(l)
        s = np.diff(ptr)
        mult = np.bincount(dofs, minlength=n)
        simple = int(np.sum(mult == 1))  # approx: DOFs in exactly one block
        lv[l] = dict(n=n, nc=nc, nnzA=case.level_A(l).nnz, nnzR=case.level_R(l).nnz,
                     F=int(np.sum(s[s > 1] * (s[s > 1] + 1) // 2)), S=int(np.sum(s[s > 1])),
                     ncx=n - simple, lst=int(np.sum(mult[mult > 1])))
    co = case.coarse()
    n0, rank = co[0].shape[0], co[2]

    def alg(step, l, acc=False):
        d = lv.get(l)
        if step == "blocks":
            return 8 * d["F"] + 16 * d["S"] + 16 * (d["S"] // 2)
        if step == "simple":
            return 20 * d["n"] + (8 * d["n"] if acc else 0) + 8 * (d["n"] - d["ncx"])
        if step == "complex":
            return d["ncx"] * (4 + 8 + 8 + 8 + (8 if acc else 0)) + 12 * d["lst"]
        if step == "residual":
            return 12 * d["nnzA"] + 4 * (d["n"] + 1) + 24 * d["n"]
        if step == "restrict":
            return 12 * d["nnzR"] + 4 * (d["nc"] + 1) + 8 * d["n"] + 8 * d["nc"]
        if step == "prolong":
            return 12 * d["nnzR"] + 4 * (d["n"] + 1) + 8 * d["nc"] + 24 * d["n"]
        if step == "coarse":
            return 8 * rank * (rank + 1) // 2 + 24 * n0
        return 0

    seq = []
    for l in range(L - 1, 0, -1):
        seq += [("blocks", l, False), ("simple", l, False), ("complex", l, False), ("residual", l, False),
                ("restrict", l, False)]
    seq.append(("coarse", 0, False))
    for l in range(1, L):
        seq += [("prolong", l, False), ("residual", l, False), ("blocks", l, True), ("simple", l, True),
                ("complex", l, True)]
    recs = ncu_records(path)
    recs = recs[-len(seq):] if len(recs) >= len(seq) else recs
    print(f"# {wl.upper()} one V-cycle, direct launches; ncu gpu__time_duration / dram bytes per kernel "
          f"(cold-cache, serialised), algorithmic bytes per SURVEY.md App. C; peak {peak:.0f} GB/s (MEASURED_PEAKS.json)\n")
    print("| # | kernel | level (n) | step | time (us) | algorithmic MB | alg. GB/s | frac | DRAM MB (ncu) |")
    print("|---|---|---|---|---|---|---|---|---|")
    tot_t = tot_a = 0.0
    for i, ((step, l, acc), r) in enumerate(zip(seq, recs)):
        t = r.get("gpu__time_duration.sum") or 0.0
        if t != t:  # nan: record without metrics
            t = 0.0
        a = alg(step, l, acc)
        dram = ((r.get("dram__bytes_read.sum") or 0) + (r.get("dram__bytes_write.sum") or 0)) / 1e6
        dram = 0.0 if dram != dram else dram
        gbs = a / (t * 1e-6) / 1e9 if t > 0 else 0.0
        n = case.level_dofs()[l]
        tot_t += t
        tot_a += a
        print(f"| {i} | `{r['name']}` | L{l} ({n}) | {step}{' (acc)' if acc else ''} | {t:.1f} | {a / 1e6:.2f} | "
              f"{gbs:.0f} | {gbs / peak:.2f} | {dram:.2f} |")
    print(f"\nTotal: {tot_t:.0f} us serialised kernel time, {tot_a / 1e9:.2f} GB algorithmic "
          f"({tot_a / (tot_t * 1e-6) / 1e9:.0f} GB/s).")


if __name__ == "__main__":
    main()
