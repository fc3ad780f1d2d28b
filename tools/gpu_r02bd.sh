#!/bin/bash
# r02bd: GPU suite on the tree + A/B of the chunk_row prefetch in the fixed / FW-pass pair kernels
# (Reddit F=32 / 128 / 256) against libalt_head.so (those kernels without it).
tag=${1:-r02bd}
out=gpurun_out
mkdir -p $out
timeout 1500 python -m pytest tests -m gpu -q > $out/${tag}_pytest.log 2>&1
echo "pytest rc=$?"; tail -2 $out/${tag}_pytest.log
for f in 32 128 256; do
  for i in 1 2; do
    timeout 600 python bench.py --f $f --steps 10 --warmup 3 --no-cpu --no-e2e > $out/${tag}_f${f}_base_$i.json 2>/dev/null
    AUTOSAGE_DEV_LIB=$PWD/libalt_head.so timeout 600 python bench.py --f $f --steps 10 --warmup 3 --no-cpu --no-e2e > $out/${tag}_f${f}_alt_$i.json 2>/dev/null
  done
done
python - $tag <<'PY'
import json, sys, glob
tag = sys.argv[1]
for f in (32, 128, 256):
    for arm in ("base", "alt"):
        rows = []
        for p in sorted(glob.glob(f"gpurun_out/{tag}_f{f}_{arm}_*.json")):
            d = json.loads(open(p).read().strip().splitlines()[-1])
            rows.append((round(d["ms_per_op"]["sddmm"], 4), d["config"]["sddmm_choice"], d["clocks"]["sm_mhz"]))
        print("F", f, arm, rows)
PY
