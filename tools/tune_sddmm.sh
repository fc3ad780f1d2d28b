#!/bin/bash
# SDDMM development sweep over F (fixed-width pass kernel vs generic chunk kernel).
cfg=${1:-reddit}
for f in 32 64 128 256; do for fixed in 1 0; do
AUTOSAGE_DEV_SDDMM_FIXED=$fixed timeout 120 python tools/profile_kernels.py --config $cfg --f $f --reps 3 \
  --sddmm sddmm:rowparallel:ft=64:rpc=4:vec=1:hubt=256,sddmm:rowparallel:ft=32:rpc=4:vec=0:hubt=256 2>&1 \
  | awk -v c=$cfg -v fx=$fixed -v f=$f '{print c, "F="f, "fixed="fx, $0}'
done; done
