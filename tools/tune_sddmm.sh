#!/bin/bash
# SDDMM development sweep: fixed-width kernel on/off across variants.
cfg=${1:-reddit}
for fixed in 1 0; do
AUTOSAGE_DEV_SDDMM_FIXED=$fixed timeout 120 python tools/profile_kernels.py --config $cfg --reps 3 \
  --sddmm sddmm:rowparallel:ft=64:rpc=4:vec=1:hubt=256,sddmm:hubsplit:ft=32:rpc=1:vec=1:hubt=256,sddmm:rowparallel:ft=64:rpc=4:vec=0:hubt=256,baseline 2>&1 \
  | awk -v c=$cfg -v fx=$fixed '{print c, "fixed="fx, $0}'
done
