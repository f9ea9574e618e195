"""Golden solve records produced by THE REFERENCE'S OWN CODE.

oracle/_ref/libimmergrid_ref.so (make -C oracle ref) is the reference's
solvers.cpp / multigrid.cpp / smoothers.cpp compiled unmodified against the
Eigen / LAPACKE stand-in of oracle/ref_shim.  This script runs its pcg
(precond = MgHierarchy::apply, tol 1e-8, zero guess) on the host-built
hierarchies of the BASELINE configs at FULL size and writes
tests/golden/reference_solves.json: iterations, the whole residual history
and checksums / samples of x.  It needs /root/reference (build time only) and
minutes of single-threaded CPU (the reference is single-threaded: C4 takes
~5 min), so it is run here and its output committed; tests/test_reference_pin.py
holds the oracle (and through tests/golden/c4_oracle.json the device) to it.

Doubles are float.hex() strings (exact round trip).

    python tests/golden/make_reference_golden.py [c1 c2 c3 c5 c4 ...]
"""
import hashlib
import json
import math
import os
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.dirname(HERE))

import numpy as np  # noqa: E402

import reference_ffi as ref  # noqa: E402
from paper_1903_10977_b200 import build_case, configs  # noqa: E402

OUT = os.path.join(HERE, "reference_solves.json")


def config_of(name):
    return {"c1": configs.c1, "c2": lambda: configs.c2(p=2, seed=configs.c2_seed()), "c3": configs.c3,
            "c4": configs.c4, "c5": configs.c5}[name]()


def record(name):
    case = build_case(config_of(name))
    h = ref.RefHierarchy(case.levels_c())
    t = time.time()
    st, x, res, it = h.pcg(case.b, tol=configs.TOL, maxit=configs.MAXIT)
    sec = time.time() - t
    h.close()
    idx = list(range(0, x.shape[0], max(1, x.shape[0] // 64)))
    return {"n": case.n, "level_dofs": case.level_dofs(),
            "b_sha256": hashlib.sha256(case.b.tobytes()).hexdigest(),
            "A_val_sha256": hashlib.sha256(np.ascontiguousarray(case.A.val).tobytes()).hexdigest(),
            "status": st, "iterations": it, "residuals": [float(v).hex() for v in res],
            "x_sha256": hashlib.sha256(np.ascontiguousarray(x).tobytes()).hexdigest(),
            "x_fsum2": math.fsum((x * x).tolist()).hex(),
            "x_sample_idx": idx, "x_sample": [float(v).hex() for v in x[idx]],
            "reference_seconds_single_thread": sec}


def main():
    names = sys.argv[1:] or ["c1", "c2", "c3", "c5", "c4"]
    out = {}
    if os.path.exists(OUT):
        with open(OUT) as f:
            out = json.load(f)
    for name in names:
        out[name] = record(name)
        print(name, "iterations", out[name]["iterations"], "seconds", round(out[name]["reference_seconds_single_thread"], 2),
              flush=True)
        with open(OUT, "w") as f:
            json.dump(out, f, indent=0)


if __name__ == "__main__":
    main()
