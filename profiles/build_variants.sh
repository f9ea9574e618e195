#!/bin/bash
# Profiling-only variant builds of the device library:
#   profiles/build_variants.sh name1:"-DFLAG ..." name2:"..." ...
# -> paper_1903_10977_b200/libig_gpu_<name>.so (load with IG_GPU_LIB=libig_gpu_<name>.so).
# Timing-only switches of spmv_psell.cuh: -DIG_DBG_SKIP=n drops one slice class from k_pspmv (1 GENERAL,
# 2 FAST / FAST2, 3 two-line, 4 every fast class, 5 FAST2M, 6 all but FAST2M, 7 all but two-line: wrong
# results, the class's share of the product's time); -DIG_PSPMV_CTA=, -DIG_PSPMV_MINB=, -DIG_F8_LD256=0.
set -e
cd "$(dirname "$0")/../paper_1903_10977_b200"
mkdir -p ../gpurun_out
for spec in "$@"; do
  name="${spec%%:*}"; flags="${spec#*:}"
  nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo -fmad=false -Xcompiler -fPIC \
    --expt-relaxed-constexpr -I../include $flags -shared -o "libig_gpu_$name.so" csrc/*.cu -lcudart \
    2> "../gpurun_out/ptxas_$name.log" &
done
wait
for spec in "$@"; do
  name="${spec%%:*}"
  echo "$name $(cuobjdump -res-usage libig_gpu_$name.so | grep -A1 'k_pspmvILi0ELb0\|k_pprolongILb0' | grep -o 'REG:[0-9]*\|STACK:[0-9]*' | paste -s -d' ')"
done
