#!/usr/bin/env python3
"""Turn gpurun_out/ ncu artefacts into the committed summaries under profiles/.

  python tools/summarize_ncu.py --tag r01 [--config reddit --f 64]

Reads
  gpurun_out/launches_<tag>.csv      ncu --metrics gpu__time_duration.sum launch list
                                     of `bench.py --steps 3 --warmup 3`
  gpurun_out/<op>_full_<tag>.ncu-rep ncu --set full of one steady-state launch
  gpurun_out/bench_<tag>.json        the bench line of the same build
Writes
  profiles/<tag>_launches.md         per-kernel share of the timed steps
  profiles/<tag>_<op>_full.md        key counters, stall mix, hottest source lines
  profiles/ncu_traffic.json          dram bytes per launch of each op's dominant
                                     kernel (bench.py -> roofline.traffic)
"""
import argparse
import csv
import json
import os
import subprocess
import sys
from collections import OrderedDict, defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "gpurun_out")
PROF = os.path.join(ROOT, "profiles")


def short(name):
    n = name.split("(")[0]
    n = n.replace("asb::<unnamed>::", "").replace("void ", "")
    return n


def launches(tag):
    path = os.path.join(OUT, f"launches_{tag}.csv")
    rows = []
    with open(path) as fh:
        lines = [ln for ln in fh if ln.startswith('"')]
    for r in csv.DictReader(lines):
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        v = float(r["Metric Value"].replace(",", ""))
        unit = r.get("Metric Unit", "ns")
        ns = v * {"ns": 1, "us": 1e3, "usecond": 1e3, "ms": 1e6, "msecond": 1e6, "nsecond": 1}.get(unit, 1)
        rows.append((int(r["ID"]), r["Kernel Name"], ns, r.get("Grid Size", ""), r.get("Block Size", "")))
    return rows


def steady_state(rows, steps):
    """The last `steps` bench steps: the launches after the final L2-flush
    fill kernel boundaries (bench.py zero_() -> elementwise fill)."""
    flush_ids = [i for i, (id_, n, *_r) in enumerate(rows) if "FillFunctor" in n or "fill_kernel" in n]
    if len(flush_ids) >= steps:
        start = flush_ids[-steps]
        return rows[start:]
    return rows


def write_launches(tag, steps, bench):
    rows = launches(tag)
    tail = steady_state(rows, steps)
    agg = OrderedDict()
    for _, name, ns, grid, block in tail:
        k = short(name)
        a = agg.setdefault(k, [0, 0.0, grid, block])
        a[0] += 1
        a[1] += ns
    total = sum(a[1] for k, a in agg.items() if "Fill" not in k and "fill" not in k)
    lines = [f"# ncu launch list ({tag})", "",
             "Command: `ncu --metrics gpu__time_duration.sum --clock-control none --csv "
             "python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu` (tools/gpu_round.sh).",
             f"All launches in the log: {len(rows)} (cold decide/probes included). Below: the last "
             f"{steps} timed steps, from the L2-flush fill that opens each step. Times are ncu's "
             "serialised, cold-cache per-launch durations; compare SHARES with bench.py's event "
             "timings, not absolutes.", "",
             "| kernel | launches | total us | share of step (excl. L2 flush) | grid | block |",
             "|---|---|---|---|---|---|"]
    for k, (n, ns, grid, block) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        share = "" if ("Fill" in k or "fill" in k) else f"{100 * ns / total:.1f}%"
        lines.append(f"| `{k}` | {n} | {ns / 1e3:.1f} | {share} | {grid} | {block} |")
    if bench:
        mo = bench.get("ms_per_op", {})
        lines += ["", "bench.py (CUDA events, same build, L2 flushed between steps): "
                  + ", ".join(f"{k} {v:.3f} ms" for k, v in mo.items()),
                  f"choices: SpMM `{bench['config'].get('spmm_choice')}`, SDDMM "
                  f"`{bench['config'].get('sddmm_choice')}`"]
    with open(os.path.join(PROF, f"{tag}_launches.md"), "w") as fh:
        fh.write("\n".join(lines) + "\n")
    return agg


def raw_metrics(rep):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    r = list(csv.reader(txt.splitlines()))
    r = [x for x in r if x]
    h, u, v = r[0], r[1], r[2]
    return {k: (x, un) for k, un, x in zip(h, u, v)}, v[h.index("Kernel Name")]


def to_bytes(val, unit):
    f = float(val.replace(",", ""))
    return f * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}.get(unit, 1)


KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput % of peak"),
    ("lts__t_sector_hit_rate.pct", "L2 hit rate"),
    ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "L2 throughput % of peak"),
    ("l1tex__throughput.avg.pct_of_peak_sustained_active", "L1/smem throughput % of peak"),
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


def write_full(tag, op, bench, cfg, f):
    rep = os.path.join(OUT, f"{op}_full_{tag}.ncu-rep")
    if not os.path.exists(rep):
        return None
    m, kname = raw_metrics(rep)
    lines = [f"# ncu --set full: {op} ({tag})", "",
             f"Kernel: `{short(kname)}`", "",
             "Command: `ncu --set full --clock-control none --import-source on -k regex:<kernel> -s 2 "
             f"-c 1 python tools/profile_kernels.py --config {cfg} --{op} <bench choice>` "
             "(tools/gpu_round.sh; one steady-state launch on the full graph).", "",
             "| counter | value |", "|---|---|"]
    for key, label in KEYS:
        if key in m:
            val, unit = m[key]
            lines.append(f"| {label} (`{key}`) | {val} {unit} |")
    stalls = []
    for k, (val, unit) in m.items():
        if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio"):
            try:
                x = float(val)
            except ValueError:
                continue
            if x > 0.05:
                stalls.append((x, k[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]))
    lines += ["", "Warp stalls (cycles per issued instruction):", "",
              "| reason | cycles |", "|---|---|"]
    lines += [f"| {n} | {x:.2f} |" for x, n in sorted(stalls, reverse=True)]
    # hottest source lines
    hot = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "ncu_lines.py"), rep, "15"],
                         capture_output=True, text=True).stdout
    lines += ["", "Hottest source lines (share of instructions / of stall samples):", "", "```",
              hot.rstrip(), "```"]
    dram = None
    if "dram__bytes_read.sum" in m and "dram__bytes_write.sum" in m:
        dram = to_bytes(*m["dram__bytes_read.sum"]) + to_bytes(*m["dram__bytes_write.sum"])
        lines += ["", f"DRAM traffic per launch: {dram / 1e9:.3f} GB (read + write)."]
    with open(os.path.join(PROF, f"{tag}_{op}_full.md"), "w") as fh:
        fh.write("\n".join(lines) + "\n")
    return dram


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--tag", required=True)
    ap.add_argument("--config", default="reddit")
    ap.add_argument("--f", type=int, default=64)
    ap.add_argument("--steps", type=int, default=3)
    a = ap.parse_args()
    os.makedirs(PROF, exist_ok=True)
    bench = None
    bp = os.path.join(OUT, f"bench_{a.tag}.json")
    if os.path.exists(bp):
        with open(bp) as fh:
            txt = [ln for ln in fh if ln.startswith("{")]
        bench = json.loads(txt[-1]) if txt else None
    if os.path.exists(os.path.join(OUT, f"launches_{a.tag}.csv")):
        write_launches(a.tag, a.steps, bench)
    tp = os.path.join(PROF, "ncu_traffic.json")
    traffic = {}
    if os.path.exists(tp):
        with open(tp) as fh:
            traffic = json.load(fh)
    for op in ("spmm", "sddmm"):
        d = write_full(a.tag, op, bench, a.config, a.f)
        if d is not None:
            traffic[f"{a.config}:F={a.f}:{op}"] = d
    with open(tp, "w") as fh:
        json.dump(traffic, fh, indent=1, sort_keys=True)
    print("wrote", sorted(os.listdir(PROF)))


if __name__ == "__main__":
    main()
