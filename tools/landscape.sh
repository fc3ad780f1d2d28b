#!/bin/bash
# Full-graph time of every shortlist variant (tools/all_variants.txt) on a config.
cfg=${1:-reddit}; f=${2:-0}
spmm=$(sed -n 1p tools/all_variants.txt); sddmm=$(sed -n 2p tools/all_variants.txt)
timeout 600 python tools/profile_kernels.py --config $cfg --f $f --reps 3 --spmm "$spmm" --sddmm "$sddmm"
