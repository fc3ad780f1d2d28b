#!/bin/bash
# r02bn: launch list (time + DRAM bytes) of the fused c5 attention after the ex change
tag=${1:-r02bn}
out=gpurun_out
rm -f $out/${tag}_att.cache
timeout 600 python tools/profile_attention.py --config reddit --fused 1 --reps 1 --cache $out/${tag}_att.cache > $out/${tag}_att0.log 2>&1
c="python tools/profile_attention.py --config reddit --fused 1 --reps 3 --cache $out/${tag}_att.cache --replay-only"
timeout 600 $c > $out/${tag}_att_plain.log 2>&1 &&
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file $out/${tag}_att_launches.csv $c > $out/${tag}_ncu_att.log 2>&1
echo "ncu rc=$?"
python - $tag <<'PY'
import csv, sys, collections
tag = sys.argv[1]
rows = [r for r in csv.reader(open(f"gpurun_out/{tag}_att_launches.csv")) if len(r) > 10]
hdr = rows[0]; data = rows[1:]
ki = hdr.index("Kernel Name"); mi = hdr.index("Metric Name"); vi = hdr.index("Metric Value"); ui = hdr.index("Metric Unit"); ii = hdr.index("ID")
per = collections.OrderedDict()
for r in data:
    per.setdefault(r[ii], {"k": r[ki]})[r[mi]] = (float(r[vi].replace(",", "")), r[ui])
agg = collections.OrderedDict()
for d in per.values():
    k = d["k"].split("(")[0].replace("void ", "")[:90]
    t = d.get("gpu__time_duration.sum", (0, ""))
    tv = t[0] * (1e-3 if t[1] in ("ns", "nsecond") else 1.0 if t[1] in ("us", "usecond") else 1e3)
    a = agg.setdefault(k, [0, 0.0]); a[0] += 1; a[1] += tv
for k, (n, us) in agg.items():
    print(f"{n:4d} launches {us/n:10.1f} us/launch  {k}")
PY
