#!/bin/bash
# SDDMM development sweep: ALU widening (MIX) on/off across variants and F.
cfg=${1:-reddit}
for f in 64 32 128; do for mix in 1 0; do
AUTOSAGE_DEV_SDDMM_MIX=$mix timeout 120 python tools/profile_kernels.py --config $cfg --f $f --reps 3 \
  --sddmm sddmm:rowparallel:ft=64:rpc=4:vec=1:hubt=256,sddmm:hubsplit:ft=32:rpc=1:vec=1:hubt=256,sddmm:rowparallel:ft=64:rpc=4:vec=0:hubt=256 2>&1 \
  | awk -v c=$cfg -v m=$mix -v f=$f '{print c, "F="f, "mix="m, $0}'
done; done
