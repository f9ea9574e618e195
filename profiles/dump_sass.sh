#!/bin/sh
# SASS listings of the V-cycle / PCG kernels (cuobjdump of the in-tree
# libig_gpu.so, sm_100a): profiles/r01_sass_<kernel>.txt.  No GPU needed.
F=${1:-paper_1903_10977_b200/libig_gpu.so}
OUT=${2:-profiles}
for k in _ZN3igk7k_pspmvILi0ELb0ELb1EEEvNS_5PSellEPKdPdS3_PKNS_8PcgStateENS_7PValTabE:k_pspmv_ax \
         _ZN3igk7k_pspmvILi1ELb0ELb1EEEvNS_5PSellEPKdPdS3_PKNS_8PcgStateENS_7PValTabE:k_pspmv_residual \
         _ZN3igk11k_as_blocksENS_8AsGroupsEPKdPdPKNS_8PcgStateE:k_as_blocks \
         _ZN3igk12k_pcg_updateEiPKdS1_PdPNS_8PcgStateES2_yy:k_pcg_update \
         _ZN3igk5k_papEiPKdS1_PNS_8PcgStateEPd:k_pap \
         _ZN3igk8k_coarseILb1ELb0EEEviiPKdPKiS2_PdPKNS_8PcgStateE:k_coarse; do
  fn=${k%%:*}; name=${k##*:}
  cuobjdump -sass "$F" | awk -v fn="$fn" 'index($0, "Function : " fn) {f=1} f && /Function :/ && !index($0, fn) {f=0} f' \
    | sed 's@ */\* 0x[0-9a-f]* \*/@@' > "$OUT/r01_sass_$name.txt"
  echo "$name: $(grep -c '^ */\*[0-9a-f]*\*/' "$OUT/r01_sass_$name.txt") instructions"
done
