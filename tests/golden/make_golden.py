"""Generate the golden fixtures in tests/golden/ from the CPU oracle.

The reference cannot be built or run here (Eigen, LAPACKE and
proj/vendor/ are absent), and it records no iteration counts or residual
digits, so the goldens come from the oracle (oracle/oracle.c), run on the
host-built hierarchies of BASELINE.json configs[0] (C1) and configs[3] (C4).
They pin the oracle/host-setup pair against regressions and give the GPU
tests full-size references without rerunning a 3-minute CPU solve.

Doubles are stored as float.hex() strings (exact round trip).

    python tests/golden/make_golden.py            # C1 only (seconds)
    python tests/golden/make_golden.py --c4       # also C4 (minutes)
"""
import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.dirname(HERE))

import numpy as np  # noqa: E402

import oracle_ffi as orc  # noqa: E402
from paper_1903_10977_b200 import build_case, configs  # noqa: E402


def hexes(a):
    return [float(v).hex() for v in np.asarray(a, np.float64)]


def solve_record(case, mode, full_x):
    st, x, res, it, sec = orc.pcg(case.levels_c(), case.b, tol=configs.TOL, maxit=configs.MAXIT, mode=mode)
    import hashlib
    import math
    # Machine-independent checksums: sha256 of the raw doubles and an exactly
    # rounded sum of squares (math.fsum); BLAS dot/sum orders vary by CPU.
    rec = {"status": st, "iterations": it, "residuals": hexes(res),
           "x_sha256": hashlib.sha256(np.ascontiguousarray(x).tobytes()).hexdigest(),
           "x_fsum2": math.fsum((x * x).tolist()).hex(),
           "x_sample_idx": list(range(0, x.shape[0], max(1, x.shape[0] // 64))),
           "cpu_seconds": sec}
    rec["x_sample"] = hexes(x[rec["x_sample_idx"]])
    if full_x:
        rec["x"] = hexes(x)
    return rec


def case_record(case):
    i = case.info
    import hashlib
    return {"n": case.n, "level_dofs": [int(i.n[k]) for k in range(case.n_levels)],
            "nnz": [int(i.nnz[k]) for k in range(case.n_levels)], "coarse_rank": int(i.coarse_rank),
            "b_sha256": hashlib.sha256(case.b.tobytes()).hexdigest(),
            "A_val_sha256": hashlib.sha256(np.ascontiguousarray(case.A.val).tobytes()).hexdigest(),
            "eta": float(i.eta).hex()}


def main():
    out = {}
    c1 = build_case(configs.c1())
    out["c1"] = {"case": case_record(c1),
                 "gpu_order": solve_record(c1, orc.GPU_ORDER, True),
                 "seq": solve_record(c1, orc.SEQ, True)}
    with open(os.path.join(HERE, "c1_oracle.json"), "w") as f:
        json.dump(out["c1"], f, indent=0)
    if "--c4" in sys.argv:
        c4 = build_case(configs.c4())
        rec = {"case": case_record(c4), "gpu_order": solve_record(c4, orc.GPU_ORDER, False),
               "seq": solve_record(c4, orc.SEQ, False)}
        with open(os.path.join(HERE, "c4_oracle.json"), "w") as f:
            json.dump(rec, f, indent=0)
    print("golden written")


if __name__ == "__main__":
    main()
