#!/bin/bash
# SpMM lane-group kernel sweep: entries in flight (U) x register cap, per config.
cfg=${1:-reddit}
for t in 4x64 4x72 4x56; do
  AUTOSAGE_DEV_SPMM_TUNE=$t timeout 120 python tools/profile_kernels.py --config $cfg --reps 3 \
    --spmm spmm:hubsplit:ft=64:rpc=4:vec=1:hubt=256,spmm:rowparallel:ft=64:rpc=4:vec=1:hubt=256 2>&1 \
    | awk -v c=$cfg -v t=$t '{print c, t, $0}'
done
