"""Summarise an ncu --csv launch list (gpu__time_duration.sum per launch)."""
import csv
import sys


def load(path):
    lines = [l for l in open(path) if l.startswith('"')]
    rows = list(csv.reader(lines))
    h = rows[0]
    ki, gi, vi = h.index("Kernel Name"), h.index("Grid Size"), h.index("Metric Value")
    out = []
    for r in rows[1:]:
        out.append((r[ki].split("(")[0].replace("void ", ""), r[gi], float(r[vi].replace(",", "")) / 1000.0))
    return out


if __name__ == "__main__":
    seq = load(sys.argv[1])
    tot = sum(t for _, _, t in seq)
    print(f"{len(seq)} launches, {tot:.1f} us total")
    agg = {}
    for n, g, t in seq:
        k = (n, g)
        agg.setdefault(k, [0, 0.0])
        agg[k][0] += 1
        agg[k][1] += t
    for (n, g), (c, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"{n:28s} grid={g:>16s} launches={c:3d} total={t:9.1f} us  share={100 * t / tot:5.1f}%")
