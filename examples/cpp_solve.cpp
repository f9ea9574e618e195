// C++ drop-in example: build a BASELINE config on the host (libig_host.so),
// hand the hierarchy across the C-ABI and solve with the reference-shaped
// immergrid_gpu::pcg / MgHierarchy (include/immergrid_gpu/solve.hpp).
//
//   ./cpp_solve [res] [levels]   (2D disc of configs[0]; defaults 32 4)
#include <cstdio>
#include <cstdlib>
#include <string>

#include "ig_host.h"
#include "immergrid_gpu/solve.hpp"

int main(int argc, char** argv) {
  const int res = argc > 1 ? std::atoi(argv[1]) : 32;
  const int levels = argc > 2 ? std::atoi(argv[2]) : 4;
  igh_config cfg;
  igh_config_default(&cfg);
  // configs.c1(): disc(0.5 + dx, 0.5 + dy, 0.4) with the seed-1 offsets.
  cfg.geometry = "disc(0.5013312315034456, 0.5049156351452541, 0.4)";
  cfg.resolution[0] = cfg.resolution[1] = res;
  cfg.levels = levels;
  igh_case* c = nullptr;
  if (igh_build(&cfg, &c) != IG_OK) {
    std::fprintf(stderr, "setup failed: %s\n", igh_last_error());
    return 2;
  }
  const ig_level* lv = nullptr;
  const ig_coarse* co = nullptr;
  int32_t nl = 0, n = 0;
  igh_levels(c, &lv, &nl, &co);
  const double* bp = igh_rhs(c, &n);
  immergrid_gpu::Vec b(bp, bp + n);
  try {
    immergrid_gpu::MgHierarchy h(lv, nl, *co);
    auto [x, rep] = immergrid_gpu::pcg(lv[nl - 1].A, b, h, 1e-8, 1000);
    std::printf("n=%d levels=%d iterations=%d final=%.6e device_seconds=%.6f\n", n, nl, rep.iterations,
                rep.residuals.back(), rep.seconds);
  } catch (const immergrid_gpu::NotConverged& e) {
    std::printf("not converged after %d iterations\n", e.report.iterations);
    igh_destroy(c);
    return 1;
  } catch (const std::exception& e) {
    std::fprintf(stderr, "error: %s\n", e.what());
    igh_destroy(c);
    return 3;
  }
  igh_destroy(c);
  return 0;
}
