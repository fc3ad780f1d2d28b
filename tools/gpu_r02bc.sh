#!/bin/bash
# e2e A/B of the short first host slice (AUTOSAGE_HOST_HEAD 8 vs 1) and an
# ncu --set full of the SDDMM pair kernel after the chunk_row prefetch.
tag=${1:-r02bc}
out=gpurun_out
mkdir -p $out
for i in 1 2; do
  for h in 8 1; do
    AUTOSAGE_HOST_HEAD=$h timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu > $out/${tag}_e2e_h${h}_$i.json 2>/dev/null
    echo "head $h run $i rc=$?"
  done
done
python - $tag <<'PY'
import json, sys, glob
tag = sys.argv[1]
for h in (8, 1):
    rows = []
    for p in sorted(glob.glob(f"gpurun_out/{tag}_e2e_h{h}_*.json")):
        d = json.loads(open(p).read().strip().splitlines()[-1])
        rows.append((round(d["e2e"]["ms_per_step"], 3), round(d["e2e"]["d2h_copy_only_ms"], 3), round(d["ms_per_step"], 3)))
    print("head", h, "(e2e ms, d2h-only ms, device ms):", rows)
PY
sd=sddmm:rowparallel:ft=32:rpc=1:vec=0:hubt=256
cmd="python tools/profile_kernels.py --config reddit --sddmm $sd --reps 3"
timeout 600 $cmd > $out/${tag}_plain_sd.log 2>&1 &&
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sddmm_pair -s 2 -c 1 -f -o $out/${tag}_sddmm $cmd > $out/${tag}_ncu_sd.log 2>&1
echo "ncu sddmm rc=$?"
if [ -f $out/${tag}_sddmm.ncu-rep ]; then
  ncu -i $out/${tag}_sddmm.ncu-rep --page raw --csv > $out/${tag}_sddmm_raw.csv 2>/dev/null
  python tools/ncu_lines.py $out/${tag}_sddmm.ncu-rep 25 > $out/${tag}_sddmm_lines.txt 2>&1
  rm -f $out/${tag}_sddmm.ncu-rep
fi
