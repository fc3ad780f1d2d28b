#!/usr/bin/env python3
"""Summaries under profiles/ from the CSVs a round-2 GPU pass leaves in
gpurun_out/ (tools/gpu_r02_profile.sh deletes the .ncu-rep files on the box
to stay under gpurun's 64 MiB merge cap, so everything here reads CSV).

  python tools/summarize_r02.py --tag r02a [--config reddit --f 64]

Reads (all optional)
  <tag>_launches_traffic.csv  ncu --metrics gpu__time_duration.sum,dram__bytes_{read,write}.sum
                              of a replayed `bench.py --steps 3 --warmup 3`
  <tag>_<name>_raw.csv        ncu --set full raw page (one row per captured kernel)
  <tag>_<name>_source.csv     ncu source page (SASS) of the same capture
  <tag>_<name>_lines.txt      tools/ncu_lines.py output (CUDA-line shares)
  <tag>_gather_roofline.txt   tools/gather_roofline output
Writes
  profiles/<tag>_launches.md            per-kernel time share + DRAM bytes of the timed steps
  profiles/ncu_traffic.json             per-op DRAM bytes per launch (bench.py roofline.traffic)
  profiles/<tag>_<name>_full.md         key counters and stall mix per captured kernel
  profiles/<tag>_gather_roofline.md, profiles/onchip_roofs.json   measured on-chip roofs
"""
import argparse
import csv
import json
import os
import re
import statistics
from collections import OrderedDict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "gpurun_out")
PROF = os.path.join(ROOT, "profiles")

UNITS = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
         "ns": 1e-9, "nsecond": 1e-9, "us": 1e-6, "usecond": 1e-6, "ms": 1e-3, "msecond": 1e-3,
         "s": 1.0, "second": 1.0}


def short(name):
    n = name.split("(")[0].replace("void ", "")
    return n.replace("asb::<unnamed>::", "").replace("(int)", "").replace("(bool)", "")


def num(val, unit):
    return float(str(val).replace(",", "")) * UNITS.get(unit, 1.0)


def csv_rows(path):
    with open(path) as fh:
        lines = [ln for ln in fh if ln.startswith('"')]
    return list(csv.DictReader(lines))


# ---------------------------------------------------------------- launches --
def launches(path):
    """[(id, kernel, {metric: value in base units})] in launch order."""
    by = OrderedDict()
    for r in csv_rows(path):
        k = int(r["ID"])
        e = by.setdefault(k, [r["Kernel Name"], {}, r.get("Grid Size", ""), r.get("Block Size", "")])
        e[1][r["Metric Name"]] = num(r["Metric Value"], r["Metric Unit"])
    return [(k, v[0], v[1], v[2], v[3]) for k, v in by.items()]


def op_of_step(kernels):
    """Split one bench step (the kernels after an L2-flush fill) into the
    SpMM op and the SDDMM op: the SDDMM starts at its first widen / sddmm
    kernel (the finite scan in front of it belongs to it)."""
    names = [short(k[1]) for k in kernels]
    first = next((i for i, n in enumerate(names) if n.startswith(("widen", "sddmm"))), len(names))
    if first > 0 and names[first - 1].startswith("finite_check"):
        first -= 1
    return ["spmm" if i < first else "sddmm" for i in range(len(names))]


def write_launches(tag, path, cfg, f, steps):
    rows = launches(path)
    fills = [i for i, r in enumerate(rows) if "FillFunctor" in r[1]]
    step_rows = []
    for j in fills[-steps:]:
        nxt = next((i for i in fills if i > j), len(rows))
        step_rows.append(rows[j + 1:nxt])
    agg = OrderedDict()
    per_op = {"spmm": [], "sddmm": []}
    for st in step_rows:
        ops = op_of_step(st)
        tot = {"spmm": [0.0, 0.0], "sddmm": [0.0, 0.0]}
        for (kid, name, m, grid, block), op in zip(st, ops):
            key = (op, short(name))
            a = agg.setdefault(key, [0, 0.0, 0.0, grid, block])
            t = m.get("gpu__time_duration.sum", 0.0)
            d = m.get("dram__bytes_read.sum", 0.0) + m.get("dram__bytes_write.sum", 0.0)
            a[0] += 1
            a[1] += t
            a[2] += d
            tot[op][0] += t
            tot[op][1] += d
        for op in per_op:
            per_op[op].append(tot[op])
    step_t = sum(a[1] for a in agg.values()) or 1.0
    n = max(len(step_rows), 1)
    lines = [f"# ncu launch list with DRAM traffic ({tag})", "",
             "Command: `ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum "
             "--clock-control none --csv python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu --cache C "
             "--replay-only` (tools/gpu_r02_profile.sh; decisions replayed, so no probes).",
             f"Last {len(step_rows)} steps (each opens with bench.py's L2-flush fill). ncu serialises "
             "launches and runs each from a cold cache: compare SHARES with bench.py's event times.", "",
             "| op | kernel | launches/step | us/launch | share of step | DRAM MB/launch | DRAM GB/s | grid | block |",
             "|---|---|---|---|---|---|---|---|---|"]
    for (op, k), (cnt, t, d, grid, block) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        lines.append(f"| {op} | `{k}` | {cnt / n:.0f} | {t / cnt * 1e6:.1f} | {100 * t / step_t:.1f}% | "
                     f"{d / cnt / 1e6:.1f} | {d / t / 1e9 if t else 0:.0f} | {grid} | {block} |")
    traffic = {}
    for op, vals in per_op.items():
        if not vals:
            continue
        t = statistics.median(v[0] for v in vals)
        d = statistics.median(v[1] for v in vals)
        traffic[op] = (t, d)
        lines.append("")
        lines.append(f"{op} op per launch: {t * 1e3:.3f} ms (ncu), DRAM {d / 1e9:.3f} GB "
                     f"({d / t / 1e9:.0f} GB/s over the ncu time)")
    with open(os.path.join(PROF, f"{tag}_launches.md"), "w") as fh:
        fh.write("\n".join(lines) + "\n")
    tp = os.path.join(PROF, "ncu_traffic.json")
    tj = {}
    if os.path.exists(tp):
        with open(tp) as fh:
            tj = json.load(fh)
    for op, (t, d) in traffic.items():
        tj[f"{cfg}:F={f}:{op}"] = {"bytes": d, "ncu_ms": t * 1e3, "source": f"profiles/{tag}_launches.md"}
    with open(tp, "w") as fh:
        json.dump(tj, fh, indent=1, sort_keys=True)
    return traffic


# -------------------------------------------------------------- full sets --
KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput % of peak"),
    ("lts__t_sector_hit_rate.pct", "L2 hit rate"),
    ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "L2 throughput % of peak"),
    ("l1tex__throughput.avg.pct_of_peak_sustained_active", "L1/smem throughput % of peak"),
    ("l1tex__t_sector_hit_rate.pct", "L1 hit rate"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "smem wavefronts"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__shared_mem_per_block_dynamic", "dynamic smem/block"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("smsp__inst_executed.sum", "warp instructions"),
    ("sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "XU pipe % (F2F)"),
    ("sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", "FP64 pipe %"),
    ("sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active", "ALU pipe %"),
    ("sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "LSU pipe %"),
]


def write_full(tag, name, what):
    raw = os.path.join(OUT, f"{tag}_{name}_raw.csv")
    if not os.path.exists(raw):
        return []
    with open(raw) as fh:
        rows = [r for r in csv.reader(fh) if r]
    hdr, units, data = rows[0], rows[1], rows[2:]
    lines = [f"# ncu --set full: {what} ({tag})", "",
             "Command: see tools/gpu_r02_profile.sh (`ncu --set full --clock-control none "
             "--import-source on`, steady-state launches on the full graph, after the same command "
             "exited 0 without ncu).", ""]
    out = []
    for r in data:
        m = {h: (v, u) for h, u, v in zip(hdr, units, r)}
        kname = short(m.get("Kernel Name", ("?", ""))[0])
        lines += [f"## `{kname}`", "", "| counter | value |", "|---|---|"]
        for key, label in KEYS:
            if key in m:
                v, u = m[key]
                lines.append(f"| {label} (`{key}`) | {v} {u} |")
        stalls = []
        for k, (v, u) in m.items():
            if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio"):
                try:
                    x = float(v)
                except ValueError:
                    continue
                if x > 0.05:
                    stalls.append((x, k[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]))
        lines += ["", "Warp stalls (cycles per issued instruction):", "", "| reason | cycles |", "|---|---|"]
        lines += [f"| {n} | {x:.2f} |" for x, n in sorted(stalls, reverse=True)[:10]]
        dram = None
        if "dram__bytes_read.sum" in m and "dram__bytes_write.sum" in m:
            dram = num(*m["dram__bytes_read.sum"]) + num(*m["dram__bytes_write.sum"])
            t = num(*m["gpu__time_duration.sum"])
            lines += ["", f"DRAM traffic per launch: {dram / 1e9:.3f} GB; {dram / t / 1e9:.0f} GB/s over "
                      f"the kernel's {t * 1e3:.3f} ms."]
        lines.append("")
        out.append((kname, dram))
    lt = os.path.join(OUT, f"{tag}_{name}_lines.txt")
    if os.path.exists(lt):
        with open(lt) as fh:
            lines += ["Hottest CUDA source lines (tools/ncu_lines.py: share of instructions / of stall "
                      "samples):", "", "```", fh.read().rstrip(), "```", ""]
    with open(os.path.join(PROF, f"{tag}_{name}_full.md"), "w") as fh:
        fh.write("\n".join(lines) + "\n")
    return out


# --------------------------------------------------------- on-chip roofs --
def write_roofs(tag):
    p = os.path.join(OUT, f"{tag}_gather_roofline.txt")
    if not os.path.exists(p):
        return
    with open(p) as fh:
        txt = fh.read()
    gathers = {}
    for m in re.finditer(r"gather (\S+)\s+U=(\d+)\s+B=(\S+): ([\d.]+) ms\s+([\d.]+) GB/s", txt):
        gathers[(m.group(1), int(m.group(2)), m.group(3))] = float(m.group(5))
    cp = re.search(r"copy 1GiB: ([\d.]+) ms\s+([\d.]+) GB/s", txt)
    l2 = {k: v for k, v in gathers.items() if "L2" in k[2]}
    hbm = {k: v for k, v in gathers.items() if "HBM" in k[2]}
    best_f64_l2 = max(v for k, v in l2.items() if k[0] != "f32-acc")
    best_f32_l2 = max(v for k, v in l2.items() if k[0] == "f32-acc")
    best_hbm = max(hbm.values())
    roofs = {
        "source": f"profiles/{tag}_gather_roofline.md (tools/gather_roofline.cu on one B200)",
        "copy_gbs": float(cp.group(2)) if cp else None,
        "gather_l2_f32acc_gbs": best_f32_l2, "gather_l2_f64_exact_gbs": best_f64_l2,
        "gather_hbm_gbs": best_hbm,
        "ops": {
            # the bit-exact SpMM / SDDMM gather one 4F-byte row per nonzero and
            # widen it to f64: their on-chip roof is the f64-exact row gather
            "spmm": {"gbs": best_f64_l2, "what": "L2-resident 256-B row gather + f32->f64 widening + DFMA "
                     "(best widening split), tools/gather_roofline.cu"},
            "sddmm": {"gbs": best_f64_l2, "what": "same row-gather roof (one Y row per nonzero)"},
        },
    }
    with open(os.path.join(PROF, "onchip_roofs.json"), "w") as fh:
        json.dump(roofs, fh, indent=1)
    lines = [f"# Measured on-chip roofs ({tag})", "",
             "`tools/gather_roofline` (nvcc -gencode arch=compute_100a,code=sm_100a -O3), one B200, "
             "CUDA events, best of 3-5. Gathers: 224,000 output rows x 512 random 256-byte B rows "
             "(F=64, 16 lanes x float4 per row), from a 60 MB B (L2-resident) or a 1 GB B (HBM).", "",
             "```", txt.rstrip(), "```", "",
             f"- HBM copy: {roofs['copy_gbs']} GB/s (read + write).",
             f"- L2-resident row gather, f32 accumulate: {best_f32_l2:.0f} GB/s of gathered rows.",
             f"- L2-resident row gather with exact f64 accumulation (F2F / ALU re-bias widening + DFMA), "
             f"best split: {best_f64_l2:.0f} GB/s -- the on-chip roof bench.py's `roofline.onchip` uses.",
             f"- HBM-resident row gather: {best_hbm:.0f} GB/s of gathered rows (reads only)."]
    with open(os.path.join(PROF, f"{tag}_gather_roofline.md"), "w") as fh:
        fh.write("\n".join(lines) + "\n")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--tag", required=True)
    ap.add_argument("--config", default="reddit")
    ap.add_argument("--f", type=int, default=64)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--full", nargs="*", default=[],
                    help="name=description pairs of <tag>_<name>_raw.csv captures")
    a = ap.parse_args()
    os.makedirs(PROF, exist_ok=True)
    lp = os.path.join(OUT, f"{a.tag}_launches_traffic.csv")
    if os.path.exists(lp):
        print("traffic", write_launches(a.tag, lp, a.config, a.f, a.steps))
    for spec in a.full:
        name, _, what = spec.partition("=")
        print(name, write_full(a.tag, name, what or name))
    write_roofs(a.tag)


if __name__ == "__main__":
    main()
