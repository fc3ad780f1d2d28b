#!/usr/bin/env python3
"""profiles/<tag>_sweep.md from a tools/sweep.py JSON.

  python tools/summarize_sweep.py gpurun_out/sweep_r01d.json r01d
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def f3(x):
    return "—" if x is None else f"{x:.3f}"


def main():
    src, tag = sys.argv[1], sys.argv[2]
    r = json.load(open(src))
    peak = r.get("peak_gbs", 6550.1)
    L = [f"# Config sweep ({tag}) — {r.get('gpu', 'B200')}", "",
         "`python tools/sweep.py` (one GPU). Times are CUDA-event medians per call after the decision is",
         "cached (device time: calls queued back to back, a 256 MB L2-flush write between them; sweeps up to",
         "r02l synchronized after every call instead); GB/s is the reference gather model",
         "(proj/src/cost.cpp:21-27) over that time, so it can exceed",
         f"HBM when the dense operand is L2-resident. `frac` = GB/s / {peak:.0f} (MEASURED_PEAKS.json).", ""]
    m = r.get("meta")
    if m:
        L += ["Run: " + ", ".join(f"{k} `{v}`" for k, v in m.items() if k != "probe_config"),
              f"probe config `{m.get('probe_config')}`", ""]
    if "c1" in r:
        c = r["c1"]
        g = c["graph"]
        L += [f"## c1 — power-law N={g['n']}, nnz={g['nnz']}, F={g['F']}", "",
              "| op | choice | ms | GB/s | frac | baseline ms |", "|---|---|---|---|---|---|"]
        for op, e in c["gpu"].items():
            L.append(f"| {op} | `{e['choice']}` | {f3(e['ms'])} | {e['gbs']:.0f} | {e['frac_hbm']:.2f} | "
                     f"{f3(e['baseline_ms'])} |")
        cpu = c.get("cpu_reference")
        if cpu:
            L += ["", f"Reference CPU library on the same graph ({cpu['cores']} host cores, {cpu['kind']}): "
                  f"{cpu['value']:.1f} GB/s for SpMM+SDDMM, {cpu['ms_per_step']:.2f} ms per step. "
                  f"{cpu['sample']}."]
        L.append("")
    if "c2" in r:
        g = r["c2"]["graph"]
        L += [f"## c2 — Reddit-shape N={g['n']}, nnz={g['nnz']}", "",
              "| F | op | choice | ms | GB/s | frac | GFLOP/s | baseline ms |",
              "|---|---|---|---|---|---|---|---|"]
        for f, ops in r["c2"]["by_F"].items():
            for op, e in ops.items():
                gf = 2.0 * g["nnz"] * int(f) / (e["ms"] * 1e-3) / 1e9  # 2*nnz*F, proj/src/cost.cpp:28
                L.append(f"| {f} | {op} | `{e['choice']}` | {f3(e['ms'])} | {e['gbs']:.0f} | "
                         f"{e['frac_hbm']:.2f} | {gf:.0f} | {f3(e['baseline_ms'])} |")
        cs = r["c2"].get("cusparse")
        if cs:
            L += ["", "cuSPARSE on the same graph via torch (fp32 accumulation, so a speed reference only — not the",
                  "reference's f64 numerics): `torch.sparse.mm` (CSR SpMM) and `torch.sparse.sampled_addmm` (CSR SDDMM).",
                  "", "| F | cuSPARSE SpMM ms | ours | cuSPARSE SDDMM ms | ours |", "|---|---|---|---|---|"]
            for f, e in cs.items():
                o = r["c2"]["by_F"][f]
                L.append(f"| {f} | {f3(e.get('spmm_ms'))} | {f3(o['spmm']['ms'])} | {f3(e.get('sddmm_ms'))} | "
                         f"{f3(o['sddmm']['ms'])} |")
        L.append("")
    if "c3" in r:
        c = r["c3"]
        g = c["graph"]
        L += [f"## c3 — Products-shape N={g['n']}, nnz={g['nnz']}, SpMM F={g['F']}, row-sharded", "",
              f"Choice `{c['choice']}`. Each rank's nnz-balanced shard is timed alone on this GPU with the full B",
              "resident (per-rank compute of a g-GPU step); the all-gather of B shards is not included (one GPU).",
              "", "| g | max-rank ms | compute speed-up | gather-model GB/s (whole job) | B bytes gathered per rank |",
              "|---|---|---|---|---|"]
        for k, e in c["by_g"].items():
            L.append(f"| {k} | {f3(e['max_rank_ms'])} | {e['compute_speedup']:.2f} | {e['gbs_total']:.0f} | "
                     f"{e['allgather_bytes_per_rank'] / 1e6:.0f} MB |")
        L.append("")
    if "c4" in r:
        L += ["## c4 — skew stressor (hubs of 1M / 250k / 60k nnz on a 1.1M-row power-law graph)", "",
              "| α | F | nnz | choice | ms | baseline ms | guardrail | replay | GB/s |",
              "|---|---|---|---|---|---|---|---|---|"]
        for e in r["c4"]:
            L.append(f"| {e['alpha']} | {e['F']} | {e['nnz']} | `{e['choice']}` | {f3(e['ms'])} | "
                     f"{f3(e['baseline_ms'])} | {'ok' if e['guardrail_ok'] else 'REGRESSED'} | "
                     f"{e['replay_source']}{'' if e['replay_same_choice'] else ' (DIFFERENT)'} | {e['gbs']:.0f} |")
        L.append("")
    if "c5" in r:
        c = r["c5"]
        g = c["graph"]
        L += [f"## c5 — CSR attention, Reddit-shape, {g['heads']} heads × F={g['F']}", "",
              f"SDDMM `{c['sddmm_choice']}`, SpMM `{c['spmm_choice']}`.", "",
              "| pipeline | ms (8 heads) | ms / head |", "|---|---|---|",
              f"| fused kernel | {c['fused_ms_8_heads']:.2f} | {c['fused_ms_8_heads'] / 8:.2f} |",
              f"| unfused (SDDMM → softmax → SpMM) | {c['unfused_ms_8_heads']:.2f} | "
              f"{c['unfused_ms_8_heads'] / 8:.2f} |", ""]
    if "bwd" in r:
        b = r["bwd"]
        g = b["graph"]
        L += [f"## bwd — backward pieces, Reddit-shape N={g['n']} nnz={g['nnz']}, F={g['F']}", "",
              "| piece | ms | note |", "|---|---|---|",
              f"| transpose (first / repeat, one-time setup) | {b['transpose_first_ms']:.1f} / {b['transpose_ms']:.1f} | host wall clock |",
              f"| permute values into Aᵀ order | {f3(b['permute_ms'])} | {b['permute_gbs']:.0f} GB/s (12 B/entry) |",
              f"| Aᵀ·dC SpMM (hubsplit ft=64) | {f3(b['spmm_t_ms'])} | {b['spmm_t_gbs']:.0f} GB/s gather-model |",
              f"| row-softmax gradient | {f3(b['softmax_bwd_ms'])} | {b['softmax_bwd_gbs']:.0f} GB/s (8(N+1) + 12·nnz) |",
              f"| spmm_csr forward + backward (torch) | {b['spmm_autograd_step_ms']:.2f} | |",
              f"| csr_attention fused forward + backward (torch) | {b['attention_autograd_step_ms']:.2f} | recompute of p |"]
        if "attention_train_step_ms" in b:
            L.append(f"| csr_attention_train forward + backward (torch) | {b['attention_train_step_ms']:.2f} | p kept from the forward |")
        L.append("")
    if "bf16" in r:
        L += ["## bf16 — SpMM with a bf16 B (as_spmm_bf16) vs f32 B, same variant", "",
              "| case | variant | f32 ms | bf16 ms | speed-up |", "|---|---|---|---|---|"]
        for k, e in r["bf16"].items():
            f32 = e.get('f32_ms', e.get('f32_staged_ms'))
            L.append(f"| {k} | `{e.get('variant', 'csr_attention staged (torch op)')}` | {f3(f32)} | "
                     f"{f3(e['bf16_ms'])} | {e['speedup']:.2f} |")
        L.append("")
    out = os.path.join(ROOT, "profiles", f"{tag}_sweep.md")
    with open(out, "w") as fh:
        fh.write("\n".join(L) + "\n")
    print("wrote", out)


if __name__ == "__main__":
    main()
