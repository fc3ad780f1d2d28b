#!/usr/bin/env python3
"""Per-CUDA-line instruction and stall-sample shares from an ncu report:
   python tools/ncu_lines.py report.ncu-rep [top]"""
import csv
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(txt.splitlines()))
hdr, out, fname = None, [], ""
for r in rows:
    if len(r) == 2 and r[0] == "File Path":
        fname = r[1].rsplit("/", 1)[-1]
    if len(r) > 5 and r[0] == "Line No":
        hdr = r
        continue
    if hdr and len(r) == len(hdr) and r[2] == "-":
        try:
            ie = int(r[hdr.index("Instructions Executed")])
            s = int(r[hdr.index("Warp Stall Sampling (All Samples)")])
        except ValueError:
            continue
        if ie or s:
            out.append((ie, s, f"{fname}:{r[0]}", r[1].strip()[:80]))
tot = sum(o[0] for o in out) or 1
ts = sum(o[1] for o in out) or 1
print(f"total warp-inst {tot}  stall samples {ts}")
for o in sorted(out, key=lambda o: -o[1])[:top]:
    print(f"{100*o[0]/tot:6.1f}% inst {100*o[1]/ts:6.1f}% stall  {o[2]:>14} {o[3]}")
