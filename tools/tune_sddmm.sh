#!/bin/bash
# SDDMM development sweep: staging buffers (NB) x ALU widening (MIX) x rows/CTA.
cfg=${1:-reddit}
for nb in 1 2; do for mix in 1 0; do
AUTOSAGE_DEV_SDDMM_NB=$nb AUTOSAGE_DEV_SDDMM_MIX=$mix timeout 120 python tools/profile_kernels.py --config $cfg --reps 3 \
  --sddmm sddmm:rowparallel:ft=64:rpc=4:vec=1:hubt=256,sddmm:rowparallel:ft=64:rpc=1:vec=1:hubt=256,sddmm:rowparallel:ft=64:rpc=16:vec=1:hubt=256 2>&1 \
  | awk -v c=$cfg -v nb=$nb -v mix=$mix '{print c, "nb="nb, "mix="mix, $0}'
done; done
