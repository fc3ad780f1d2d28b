#!/bin/bash
# r02bf: Products SpMM with narrow feature tiles swept in tile-major order
# (AUTOSAGE_DEV_SPMM_TW) so the B column slice in flight fits the L2.
tag=${1:-r02bf}
out=gpurun_out
mkdir -p $out
AUTOSAGE_DEV_SPMM_TW=8 timeout 900 python bench.py --config products --steps 5 --warmup 3 --no-e2e > $out/${tag}_tw8_parity.json 2> $out/${tag}_tw8_parity.err
echo "tw8 parity rc=$?"
for tw in 0 8 16 24 32 48; do
  AUTOSAGE_DEV_SPMM_TW=$tw timeout 600 python bench.py --config products --steps 10 --warmup 3 --no-cpu --no-e2e > $out/${tag}_tw${tw}.json 2>/dev/null
  echo "tw $tw rc=$?"
done
python - $tag <<'PY'
import json, sys
tag = sys.argv[1]
d = json.loads(open(f"gpurun_out/{tag}_tw8_parity.json").read().strip().splitlines()[-1])
print("tw8 parity", d.get("parity"), d["ms_per_op"])
for tw in (0, 8, 16, 24, 32, 48):
    try:
        d = json.loads(open(f"gpurun_out/{tag}_tw{tw}.json").read().strip().splitlines()[-1])
        print("tw", tw, round(d["ms_per_op"]["spmm"], 3), d["config"]["spmm_choice"], d["clocks"]["sm_mhz"])
    except Exception as e:
        print("tw", tw, "failed", e)
PY
