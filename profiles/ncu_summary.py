"""Text summary of one `ncu --set full --import-source on` capture of k_pspmv
(profiles/run_round_bench.sh): headline metrics from the raw page and the L1
tag requests / stall samples per CUDA source line from the source page.

  python profiles/ncu_summary.py gpurun_out/pspmv_raw.csv gpurun_out/pspmv_src.csv > profiles/r02_ncu_pspmv_c4.txt
"""
import csv
import sys


def num(x):
    try:
        return float(x.replace(",", ""))
    except ValueError:
        return 0.0


def raw(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    hdr, units, vals = rows[0], rows[1], rows[2]
    return {h: (v, u) for h, u, v in zip(hdr, units, vals)}


def lines(path):
    cur, hdr, agg = None, None, {}
    for r in csv.reader(open(path)):
        if len(r) == 2 and r[0] == "File Path":
            cur = r[1].split("/")[-1]
            continue
        if len(r) > 5 and r[0] == "Line No":
            hdr = r
            continue
        if hdr is None or len(r) < len(hdr) - 2 or r[2] != "-":
            continue
        tag, smp, ins = hdr.index("L1 Tag Requests Global"), hdr.index("# Samples"), hdr.index("Instructions Executed")
        a = agg.setdefault((cur, int(r[0])), [0.0, 0.0, 0.0, r[1].strip()])
        a[0] += num(r[tag])
        a[1] += num(r[smp])
        a[2] += num(r[ins])
    return agg


def main():
    m = raw(sys.argv[1])
    def g(k):  # exact name, else the first metric whose name ends with it (section-prefixed duplicates)
        if k in m:
            return num(m[k][0])
        for h, (v, _) in m.items():
            if h.endswith(k) and v != "":
                return num(v)
        return 0.0
    print("# ncu --set full --import-source on --clock-control none -k regex:k_pspmv -s 1 -c 1 python profiles/profile_c4.py spmv")
    print("# (C4 finest A p, 1,999,453 rows, 240.5 M nnz; one launch, cold replay -- the live time is bench.py's)")
    print("# Kernel:", m["Kernel Name"][0])
    rd, wr = g("dram__bytes_read.sum"), g("dram__bytes_write.sum")
    scale = {"Mbyte": 1.0, "Gbyte": 1e3, "Kbyte": 1e-3, "byte": 1e-6}
    rd *= scale.get(m["dram__bytes_read.sum"][1], 1.0)
    wr *= scale.get(m["dram__bytes_write.sum"][1], 1.0)
    wf, cyc = g("l1tex__data_pipe_lsu_wavefronts.avg"), g("sm__cycles_active.avg")
    if wf == 0.0:  # the triage section's raw count is "no data" in some captures: derive it from the throughput fraction
        wf = g("l1tex__throughput.avg.pct_of_peak_sustained_active") / 100.0 * cyc
    out = [
        ("gpu__time_duration.sum", f"{g('gpu__time_duration.sum'):.2f} {m['gpu__time_duration.sum'][1]}"),
        ("dram__bytes_read.sum", f"{rd:.2f} MB"),
        ("dram__bytes_write.sum", f"{wr:.2f} MB"),
        ("dram traffic per launch", f"{rd + wr:.2f} MB"),
        ("l1tex__data_pipe_lsu_wavefronts.avg (per SM)", f"{wf:,.0f} over sm__cycles_active.avg {cyc:,.0f} -> {100 * wf / cyc:.1f} % (binding unit)"),
        ("l1tex__throughput.avg.pct_of_peak_sustained_active", f"{g('l1tex__throughput.avg.pct_of_peak_sustained_active'):.1f} %"),
        ("l1tex__t_sector_hit_rate.pct", f"{g('l1tex__t_sector_hit_rate.pct'):.1f} %"),
        ("lts__t_sector_hit_rate.pct", f"{g('lts__t_sector_hit_rate.pct'):.1f} %"),
        ("sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", f"{g('sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active'):.1f} %"),
        ("sm__inst_executed_pipe_adu.avg.pct_of_peak_sustained_active", f"{g('sm__inst_executed_pipe_adu.avg.pct_of_peak_sustained_active'):.1f} %   (indexed constant-bank value reads)"),
        ("smsp__issue_active.avg.pct_of_peak_sustained_active", f"{g('smsp__issue_active.avg.pct_of_peak_sustained_active'):.1f} %"),
        ("sm__warps_active.avg.pct_of_peak_sustained_active", f"{g('sm__warps_active.avg.pct_of_peak_sustained_active'):.1f} %   (64 registers: 50 % theoretical)"),
        ("smsp__inst_executed.sum", f"{g('smsp__inst_executed.sum'):,.0f}"),
    ]
    for k, v in out:
        print(f"{k:62s} {v}")
    if len(sys.argv) > 2:
        agg = lines(sys.argv[2])
        tot = [sum(a[i] for a in agg.values()) or 1.0 for i in range(3)]
        print(f"# Per CUDA source line (--page source --print-source cuda,sass): {tot[0]:,.0f} L1 tag requests, "
              f"{tot[1]:,.0f} stall samples, {tot[2]:,.0f} warp instructions")
        print("# tags %  samples %  inst %   file:line  source")
        top = sorted(agg.items(), key=lambda kv: -(kv[1][0] / tot[0] + kv[1][1] / tot[1]))[:24]
        for (f, ln), a in top:
            print(f"  {100 * a[0] / tot[0]:5.1f}    {100 * a[1] / tot[1]:5.1f}    {100 * a[2] / tot[2]:5.1f}   {f}:{ln}  {a[3][:100]}")


if __name__ == "__main__":
    main()
