#!/bin/bash
# A/B two builds of the library on the bench (alternating runs, no profiler):
#   gpurun -- 'bash tools/ab_lib.sh <tag> <alt.so> [configs...]'
tag=$1; alt=$2; shift 2
cfgs=${@:-reddit}
out=gpurun_out
for cfg in $cfgs; do
  for i in 1 2 3; do
    timeout 600 python bench.py --config $cfg --steps 20 --warmup 5 --no-cpu --no-e2e > $out/${tag}_${cfg}_base_$i.json 2>/dev/null
    AUTOSAGE_DEV_LIB=$PWD/$alt timeout 600 python bench.py --config $cfg --steps 20 --warmup 5 --no-cpu --no-e2e > $out/${tag}_${cfg}_alt_$i.json 2>/dev/null
  done
done
python - "$tag" $cfgs <<'PY'
import json, sys, glob
tag = sys.argv[1]
for cfg in sys.argv[2:]:
    for arm in ("base", "alt"):
        rows = []
        for p in sorted(glob.glob(f"gpurun_out/{tag}_{cfg}_{arm}_*.json")):
            try:
                d = json.loads(open(p).read().strip().splitlines()[-1])
                rows.append((d["ms_per_step"], d["ms_per_op"]["spmm"], d["ms_per_op"]["sddmm"], d["clocks"]["sm_mhz"]))
            except Exception as e:
                rows.append(str(e))
        print(cfg, arm, rows)
PY
