#!/bin/bash
# r02bo: softmax chain kernel streaming 8 chunks ahead (tree) vs one chunk ahead (libalt_chain1.so):
# c5 fused / unfused attention and the GPU softmax + attention tests
tag=${1:-r02bo}
out=gpurun_out
timeout 900 python -m pytest tests -m gpu -q -k "softmax or attention or half or backward or torch" > $out/${tag}_pytest.log 2>&1
echo "pytest rc=$?"; tail -2 $out/${tag}_pytest.log
for i in 1 2; do
  timeout 900 python tools/sweep.py --cases c5 --out $out/${tag}_tree_$i.json > /dev/null 2>&1
  AUTOSAGE_DEV_LIB=$PWD/libalt_chain1.so timeout 900 python tools/sweep.py --cases c5 --out $out/${tag}_alt_$i.json > /dev/null 2>&1
done
python - $tag <<'PY'
import json, sys
tag = sys.argv[1]
for arm in ("tree", "alt"):
    for i in (1, 2):
        try:
            c = json.load(open(f"gpurun_out/{tag}_{arm}_{i}.json"))["c5"]
            print(arm, i, "fused", round(c["fused_ms_8_heads"], 2), "unfused", round(c["unfused_ms_8_heads"], 2))
        except Exception as e:
            print(arm, i, "failed", e)
PY
