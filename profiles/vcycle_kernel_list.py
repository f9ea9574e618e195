"""Per-kernel list of ONE V-cycle from an ncu launch list of
`profiles/profile_c4.py vcycle2` (two V-cycles, direct launches; the second
is tabulated): kernel, level, step, ncu time and DRAM bytes.  Levels are
attributed from the launch order (descent: smoother, residual, restriction
per level; coarse; ascent: prolongation, residual, smoother).

  python profiles/vcycle_kernel_list.py gpurun_out/vc_c4.csv 6 > profiles/r02_vcycle_kernels_c4.md
"""
import csv
import sys


def records(path):
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
            sc = {"ns": 1e-3, "us": 1.0, "ms": 1e3, "byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3}
            recs[k][d["Metric Name"]] = float(v) * sc.get(d["Metric Unit"], 1.0)
    return [recs[k] for k in order]


def main():
    path, L = sys.argv[1], int(sys.argv[2])
    ks = records(path)
    ks = ks[len(ks) // 2:]
    level, down = L - 1, True
    out, tot = [], 0.0
    for r in ks:
        n = r["name"]
        if n.startswith("k_coarse"):
            step, lev, down = "coarse", 0, False
            level = 0
        elif down:
            lev = level
            if "pspmv<1" in n or "spmv_grp<1" in n:
                step = "residual"
            elif "pspmv<0" in n or "spmv_grp<0" in n:
                step = "restrict"
                level -= 1
            else:
                step = "smoother"
        else:
            if "prolong" in n:
                level += 1
                step = "prolong"
            elif "pspmv<1" in n or "spmv_grp<1" in n:
                step = "residual"
            else:
                step = "smoother (acc)"
            lev = level
        t = r.get("gpu__time_duration.sum", 0.0)
        dram = r.get("dram__bytes_read.sum", 0.0) + r.get("dram__bytes_write.sum", 0.0)
        tot += t
        out.append(f"| `{n}` | L{lev} | {step} | {t:.1f} | {dram:.2f} |")
    print("# C4 one V-cycle (second of two, direct launches), ncu gpu__time_duration and DRAM bytes per kernel\n"
          "# (--cache-control none --clock-control none: warm L2, serialised, no PDL overlap; the graph-launched\n"
          "# V-cycle takes ~750 us, profiles/level_costs.py)\n")
    print("| kernel | level | step | time (us) | DRAM MB |")
    print("|---|---|---|---|---|")
    print("\n".join(out))
    print(f"\nTotal: {tot:.0f} us serialised kernel time over {len(ks)} kernels.")


if __name__ == "__main__":
    main()
