#!/bin/bash
# r02bj: SDDMM pair-kernel shared-memory layout A/B, three arms alternating:
#   tree  = X rows padded off each other's banks + per-warp regions rounded to 128 B
#   round = per-warp regions rounded to 128 B only (libalt_round.so)
#   head  = the committed layout (libalt_head.so)
tag=${1:-r02bj}
out=gpurun_out
for cfg in reddit products c1; do
  for i in 1 2; do
    for arm in tree round head; do
      lib=""; [ $arm != tree ] && lib="AUTOSAGE_DEV_LIB=$PWD/libalt_$arm.so"
      env $lib timeout 600 python bench.py --config $cfg --steps 10 --warmup 3 --no-cpu --no-e2e > $out/${tag}_${cfg}_${arm}_$i.json 2>/dev/null
    done
  done
done
python - $tag <<'PY'
import json, sys, glob
tag = sys.argv[1]
for cfg in ("reddit", "products", "c1"):
    for arm in ("tree", "round", "head"):
        rows = []
        for p in sorted(glob.glob(f"gpurun_out/{tag}_{cfg}_{arm}_*.json")):
            d = json.loads(open(p).read().strip().splitlines()[-1])
            rows.append((round(d["ms_per_op"]["sddmm"], 4), d["clocks"]["sm_mhz"]))
        print(cfg, arm, rows)
PY
