#!/bin/bash
# compute-sanitizer over the small-case GPU tests (every kernel family:
# SpMV layouts, smoothers additive / multiplicative, coarse solve, PCG and
# Richardson graphs and host loops, Galerkin SpGEMM, block factorisation,
# pstrf, assembly) and over smoke().  Run on the GPU box from the repo root:
#   bash profiles/sanitize.sh   -> gpurun_out/sanitize_*.log
set -u
OUT=${OUT:-gpurun_out}
mkdir -p "$OUT"
CS="compute-sanitizer --print-limit 20 --error-exitcode 99"
TESTS="tests/test_gpu_parity.py tests/test_gpu_layouts.py tests/test_gpu_multiplicative.py tests/test_gpu_blockfac.py \
tests/test_gpu_galerkin.py tests/test_gpu_assembly.py tests/test_richardson.py tests/test_gpu_boundary.py"
run() {
  local tool=$1; shift
  echo "== $tool: $*" >> "$OUT/sanitize_$tool.log"
  timeout 3000 $CS --tool "$tool" "$@" >> "$OUT/sanitize_$tool.log" 2>&1
  echo "rc=$?" >> "$OUT/sanitize_$tool.log"
}
rm -f "$OUT"/sanitize_*.log
# memcheck: the small cases of every GPU test file (full-size C2-C5 excluded for time)
run memcheck python -m pytest $TESTS -m gpu -q -x -k "not full_size and not c4 and not c3_small and not thb and not d3_48" -p no:cacheprovider
# racecheck / synccheck / initcheck: the solve path (smoke: C1 through the graph and the host loop)
run racecheck python -c "import __graft_entry__ as g; g.smoke()"
run synccheck python -c "import __graft_entry__ as g; g.smoke()"
run initcheck python -c "import __graft_entry__ as g; g.smoke()"
for t in memcheck racecheck synccheck initcheck; do
  echo "$t: $(grep -c 'ERROR SUMMARY: 0 errors' "$OUT/sanitize_$t.log") clean runs, $(grep -E 'ERROR SUMMARY: [1-9]' "$OUT/sanitize_$t.log" | head -3 | tr '\n' ' '); $(grep '^rc=' "$OUT/sanitize_$t.log" | tr '\n' ' ')"
done
