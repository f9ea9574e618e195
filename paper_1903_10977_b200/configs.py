"""The BASELINE.json workloads as host-setup configurations (SURVEY.md §8d,
Appendix B).  Seeded with the reference's splitmix64 Rng (common.hpp:43-58).

Deviations from the config text, all forced by the reference:
  * "Nitsche Dirichlet" -> penalty Dirichlet with beta = 2/h (D1; the reference
    implements only the penalty method, assembly.cpp:106-131);
  * additive Schwarz with gamma = 1/max N_K (D4);
  * levels for C3/C4 chosen so the coarsest grid is 4 cells per axis (D7).
C5 uses the THB space (host/thb.cpp) with a hierarchy that follows the
refinement levels (the reference's Algorithm-2 coarsening).
"""
from __future__ import annotations

from . import CaseConfig, SmootherConfig, seed_offsets

TOL = 1e-8
MAXIT = 1000


class _Rng:
    """splitmix64 (common.hpp:43-58)."""

    M = (1 << 64) - 1

    def __init__(self, seed: int):
        self.s = seed

    def uniform(self, a: float = 0.0, b: float = 1.0) -> float:
        self.s = (self.s + 0x9E3779B97F4A7C15) & self.M
        z = self.s
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & self.M
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & self.M
        z ^= z >> 31
        return a + (b - a) * ((z >> 11) * 2.0 ** -53)


def disc_geometry(seed: int = 1, r: float = 0.4) -> str:
    dx, dy, _ = seed_offsets(seed)
    return f"disc({0.5 + dx!r}, {0.5 + dy!r}, {r!r})"


def c1(threads: int = 0) -> CaseConfig:
    """2D disc, 32x32, p=2 B-splines, 4 levels (configs[0])."""
    return CaseConfig(geometry=disc_geometry(1), dim=2, resolution=(32, 32, 1), degree=2, levels=4,
                      smoother=SmootherConfig("additive-schwarz"), threads=threads)


def c2(p: int = 2, seed: int = 1, threads: int = 0) -> CaseConfig:
    """2D disc, 512x512, p in 1..4, 8 levels (configs[1]); `seed` from c2_seed()."""
    return CaseConfig(geometry=disc_geometry(seed), dim=2, resolution=(512, 512, 1), degree=p, levels=8,
                      smoother=SmootherConfig("additive-schwarz"), threads=threads)


def c2_seed(max_seed: int = 200) -> int:
    """Smallest seed s >= 1 whose min cut fraction eta < 1e-4 (App. B)."""
    import ctypes as C
    from . import _ffi
    for s in range(1, max_seed + 1):
        cfg = c2(2, s).to_c()
        eta, cut, n = C.c_double(), C.c_int64(), C.c_int32()
        _ffi.host().igh_eta(C.byref(cfg), C.byref(eta), C.byref(cut), C.byref(n))
        if eta.value < 1e-4:
            return s
    raise RuntimeError("no seed with eta < 1e-4")


def c3_geometry(seed: int = 1, holes: int = 64) -> str:
    rng = _Rng(seed)
    acc = []
    while len(acc) < holes:
        cx, cy = rng.uniform(0.05, 0.95), rng.uniform(0.05, 0.95)
        r = rng.uniform(0.02, 0.05)
        if all(((cx - x) ** 2 + (cy - y) ** 2) ** 0.5 - r - rr >= 0.01 for x, y, rr in acc):
            acc.append((cx, cy, r))
    discs = ", ".join(f"disc({x!r}, {y!r}, {r!r})" for x, y, r in acc)
    return f"complement(union({discs}))"


def c3(threads: int = 0) -> CaseConfig:
    """2D perforated plate, 1024x1024, p=2, 9 levels, Dirichlet on holes and box edges (configs[2])."""
    return CaseConfig(geometry=c3_geometry(1), dim=2, resolution=(1024, 1024, 1), degree=2, levels=9,
                      dirichlet_box_sides=True, smoother=SmootherConfig("additive-schwarz"), threads=threads)


def c4_geometry(seed: int = 1, r: float = 0.3) -> str:
    dx, dy, dz = seed_offsets(seed)
    return f"complement(sphere({0.5 + dx!r}, {0.5 + dy!r}, {0.5 + dz!r}, {r!r}))"


def c4(res: int = 128, levels: int = 6, threads: int = 0, seed: int = 1) -> CaseConfig:
    """3D cube minus sphere, 128^3, p=2, 6 levels (configs[3], the north star).
    Dirichlet on the sphere only (cube faces natural).  Cut-cell quadrature
    depth 2 (octree) in 3D; see DESIGN.md.  `seed` draws the sphere offset
    (the mesh/cut-independence family, tests/test_gpu_mesh_independence.py)."""
    return CaseConfig(geometry=c4_geometry(seed), dim=3, resolution=(res, res, res), degree=2, levels=levels,
                      quad_depth=2, dirichlet_box_sides=False, smoother=SmootherConfig("additive-schwarz"),
                      threads=threads)


def c5(threads: int = 0, base: int = 128, levels: int = 6) -> CaseConfig:
    """2D THB (configs[4]): p=2, base 128^2 on [0,1]^2, two passes of local
    dyadic refinement on elements within 0.05 of the circle r=0.4 centred at
    (0.5+d, 0.5+d) (the same seed-1 delta on both axes as
    the config text), Dirichlet on the circle, hierarchy following the
    refinement levels (coarsen keeps the 2 local levels, base down to 4)."""
    d = seed_offsets(1)[0]
    c = 0.5 + d
    return CaseConfig(geometry=f"disc({c!r}, {c!r}, 0.4)", dim=2, resolution=(base, base, 1), family="thb",
                      degree=2, levels=levels, smoother=SmootherConfig("additive-schwarz"), threads=threads,
                      refine_passes=2, refine_circle=(c, c, 0.4), refine_dist=0.05)


def c4_levels(res: int) -> int:
    """Levels so the coarsest grid is 4 cells per axis (D7): 16 -> 3 ... 128 -> 6."""
    return max(1, res.bit_length() - 2)


CONFIGS = {"c1": c1, "c2": c2, "c3": c3, "c4": c4, "c5": c5}
