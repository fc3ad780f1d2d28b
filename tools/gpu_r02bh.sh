#!/bin/bash
# r02bh: e2e A/B of the double-buffered host-pipeline output staging (base)
# against the single-buffered library (alt, libalt_e2e.so), same bench.py:
# pipelined (k steps back to back) and synchronized-per-step timings.
tag=${1:-r02bh}
out=gpurun_out
for i in 1 2 3; do
  timeout 600 python bench.py --no-cpu > $out/${tag}_base_$i.json 2>/dev/null
  AUTOSAGE_DEV_LIB=$PWD/libalt_e2e.so timeout 600 python bench.py --no-cpu > $out/${tag}_alt_$i.json 2>/dev/null
done
python - $tag <<'PY'
import json, sys, glob
tag = sys.argv[1]
for arm in ("base", "alt"):
    for p in sorted(glob.glob(f"gpurun_out/{tag}_{arm}_*.json")):
        d = json.loads(open(p).read().strip().splitlines()[-1]); e = d["e2e"]
        print(arm, "pipelined", round(e["ms_per_step"], 3), "synced", round(e["ms_per_step_synced"], 3),
              "d2h-only", round(e["d2h_copy_only_ms"], 3), "match", e.get("outputs_vs_device_path"))
PY
