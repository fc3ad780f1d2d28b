#!/bin/bash
for rep in 1 2; do
for t in default 8x96 8x80 6x80 8x64 8x128 4x72; do
  if [ $t = default ]; then timeout 300 python tools/ab_c4_tune.py; else AUTOSAGE_DEV_SPMM_TUNE=$t timeout 300 python tools/ab_c4_tune.py; fi
done
done
