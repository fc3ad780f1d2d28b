#!/bin/bash
# SDDMM: pair kernel (64-entry chunks) vs fixed kernel (32-entry), across F.
cfg=${1:-reddit}
for f in 64 128 256; do for pair in 0 1; do
AUTOSAGE_DEV_SDDMM_PAIR=$pair timeout 120 python tools/profile_kernels.py --config $cfg --f $f --reps 3 \
  --sddmm sddmm:rowparallel:ft=64:rpc=4:vec=1:hubt=256,sddmm:rowparallel:ft=32:rpc=4:vec=0:hubt=256 2>&1 \
  | awk -v c=$cfg -v p=$pair -v f=$f '{print c, "F="f, "pair="p, $0}'
done; done
