"""CPU-side statistics of the pattern-SELL run structure of a level operator
(no GPU): run-length distribution of identical consecutive rows, value-sequence
classes, segment structure.  python profiles/layout_stats.py [workload] [res]"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def row_hash(words, ptr, salt):
    n = len(ptr) - 1
    lens = np.diff(ptr)
    pos = np.arange(len(words), dtype=np.uint64) - np.repeat(ptr[:-1].astype(np.uint64), lens)
    with np.errstate(over="ignore"):
        w = (words.astype(np.uint64) + np.uint64(salt)) * (np.uint64(2) * pos + np.uint64(1)) * np.uint64(0x9E3779B97F4A7C15)
        w ^= w >> np.uint64(29)
        w *= np.uint64(0xBF58476D1CE4E5B9)
        h = np.add.reduceat(w, ptr[:-1].astype(np.int64)) if n else np.zeros(0, np.uint64)
        h = h + lens.astype(np.uint64) * np.uint64(0x94D049BB133111EB)
    return h


def main():
    from paper_1903_10977_b200 import build_case, configs
    wl = sys.argv[1] if len(sys.argv) > 1 else "c4"
    if wl == "c4":
        res = int(sys.argv[2]) if len(sys.argv) > 2 else 128
        cfg = configs.c4(res=res, levels=configs.c4_levels(res))
    else:
        cfg = configs.CONFIGS[wl]()
    case = build_case(cfg)
    A = case.A.to_scipy().tocsr()
    ptr, col, val = A.indptr.astype(np.int64), A.indices.astype(np.int64), A.data
    n = A.shape[0]
    lens = np.diff(ptr)
    rows = np.repeat(np.arange(n, dtype=np.int64), lens)
    hv = row_hash(val.view(np.uint64), ptr, 1)
    ho = row_hash((col - rows).astype(np.int64).view(np.uint64), ptr, 2)
    # segment structure: lengths of maximal consecutive-column runs
    newseg = np.ones(len(col), dtype=bool)
    newseg[1:] = (col[1:] != col[:-1] + 1) | (rows[1:] != rows[:-1])
    segid = np.cumsum(newseg) - 1
    seglen = np.bincount(segid)
    segrow = rows[newseg]
    sptr = np.zeros(n + 1, np.int64)
    np.cumsum(np.bincount(segrow, minlength=n), out=sptr[1:])
    hs = row_hash(seglen.astype(np.uint64), sptr, 3)  # structure hash (segment lengths)
    brk = np.ones(n, dtype=bool)
    brk[1:] = (hv[1:] != hv[:-1]) | (ho[1:] != ho[:-1])
    starts = np.flatnonzero(brk)
    rl = np.diff(np.append(starts, n))
    print(f"n={n} nnz={len(col)} runs={len(starts)}")
    edges = [1, 2, 4, 8, 16, 32, 64, 96, 120, 128, 1 << 30]
    for a, b in zip(edges[:-1], edges[1:]):
        m = (rl >= a) & (rl < b)
        print(f"  run length [{a},{b}): {m.sum():8d} runs, {rl[m].sum():9d} rows ({100.0 * rl[m].sum() / n:5.1f} %)")
    run_of = np.repeat(np.arange(len(starts)), rl)
    rlen_row = rl[run_of]
    for name, mask in (("rows in runs >= 8", rlen_row >= 8), ("rows in runs < 8", rlen_row < 8)):
        idx = np.flatnonzero(mask)
        print(f"{name}: {len(idx)} rows")
        for label, h in (("value", hv), ("value+structure", hv ^ (hs * np.uint64(3))), ("structure", hs), ("offsets", ho)):
            u, c = np.unique(h[idx], return_counts=True)
            o = np.argsort(-c)
            top = c[o][:8]
            cum = np.cumsum(c[o])
            print(f"  distinct {label:16s}: {len(u):8d}; top classes {top.tolist()}; classes covering 50/80/90/95 %: "
                  f"{[int(np.searchsorted(cum, f * len(idx)) + 1) for f in (0.5, 0.8, 0.9, 0.95)]}")
    # rows in runs >= 8 with the dominant value sequence: run-length distribution
    idx = np.flatnonzero(rlen_row >= 8)
    u, c = np.unique(hv[idx], return_counts=True)
    dom = u[np.argmax(c)]
    rmask = (hv[starts] == dom) & (rl >= 8)
    print(f"dominant value sequence: {c.max()} rows in {rmask.sum()} runs >= 8; run-length histogram:")
    for a, b in zip(edges[3:-1], edges[4:]):
        m = rmask & (rl >= a) & (rl < b)
        print(f"  [{a},{b}): {m.sum():7d} runs {rl[m].sum():9d} rows")
    # dominant value sequence among ALL rows (including short runs)
    print(f"rows with the dominant value sequence overall: {(hv == dom).sum()} ; in runs < 8: {((hv == dom) & (rlen_row < 8)).sum()}")
    np.savez_compressed(os.path.join(ROOT, "gpurun_out", f"layout_{wl}.npz"), hv=hv, ho=ho, hs=hs, rl=rl, starts=starts, lens=lens)


if __name__ == "__main__":
    main()
