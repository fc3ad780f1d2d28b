"""autosage-bench for B200: the reference's measurement CLI over the GPU library.

    python -m paper_2511_17594_b200.cli <subcommand> [options]

Mirrors proj/tools/autosage_bench.cpp: the same subcommands
(gen, bench, sweep-split, ablate-vec, attention, replay), option names, CSV
columns, `<csv>.meta.json` sidecar fields and exit codes (0 ok, 1 usage, 2 I/O
or cache, 3 replay miss; autosage_bench.cpp:38-41, :733-750).

What differs, on purpose:
- times are CUDA-event medians of `--iters` runs after `--warmups` (the
  reference's bench_median_ms, autosage_bench.cpp:65-79, times host calls with
  steady_clock); operands stay resident on the GPU;
- dense operands come from the library's deterministic generator
  (`fill_uniform`, U(-1,1), same seed arithmetic as seeded_dense,
  autosage_bench.cpp:55-63), not libstdc++'s mt19937_64 stream;
- `gen er|hubskew|hubfixed` draw their own streams (numpy PCG64) with the
  reference generators' shapes (src/generate.cpp:41-132); `gen powerlaw` is the
  device power-law generator the BASELINE configs use.  ASCR files
  (src/io.cpp:48-93) interoperate both ways.
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

import numpy as np

import paper_2511_17594_b200 as asb

EXIT_OK, EXIT_USAGE, EXIT_IO, EXIT_REPLAY_MISS = 0, 1, 2, 3  # autosage_bench.cpp:38-41


def dataset_name(path: str) -> str:  # autosage_bench.cpp:42-44
    return os.path.splitext(os.path.basename(path))[0]


def round3(v: float) -> float:
    return float(np.round(v * 1000.0) / 1000.0)


def fmt3(v: float) -> str:
    return "%.3f" % v


def seeded_dense(rows: int, cols: int, seed: int):
    import torch
    return torch.from_numpy(asb.fill_uniform(rows * cols, seed, (rows, cols))).cuda()


def median_ms(run, iters: int, warmups: int) -> float:
    """Median (lower) of `iters` CUDA-event timings after `warmups` runs."""
    import torch
    for _ in range(warmups):
        run()
    times = []
    for _ in range(max(iters, 1)):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        run()
        e1.record()
        e1.synchronize()
        times.append(e0.elapsed_time(e1))
    times.sort()
    return times[(len(times) - 1) // 2]


def env_snapshot() -> dict:
    return {k: v for k, v in sorted(os.environ.items()) if k.startswith("AUTOSAGE_")}


def versions() -> dict:
    """The paper's sidecar extras: Torch / CUDA versions and the
    GPU's SM architecture, beside the reference's fields."""
    import platform
    out = {"python": platform.python_version()}
    try:
        import torch
        out["torch"] = torch.__version__
        out["cuda_runtime"] = torch.version.cuda
        if torch.cuda.is_available():
            p = torch.cuda.get_device_properties(torch.cuda.current_device())
            out["gpu"] = p.name
            out["sm"] = f"sm_{p.major}{p.minor}"
            out["sms"] = p.multi_processor_count
    except Exception:  # noqa: BLE001 -- the sidecar is best-effort metadata
        pass
    return out


def write_sidecar(csv_path: str, command: str, dp: asb.DeviceProfile, config: dict) -> None:
    """autosage_bench.cpp:144-164."""
    meta = {"artifact_version": dp.device_sig.rsplit("|", 1)[-1],
            "toolchain": asb.toolchain_tag(), "command": command,
            "timestamp_unix": int(time.time()),
            "device": {"device_sig": dp.device_sig, "bw_eff_bytes_per_s": dp.bw_eff,
                       "flops_eff_per_s": dp.flops_eff, "cores": dp.cores},
            "config": config, "env": env_snapshot(), "versions": versions()}
    path = csv_path + ".meta.json"
    try:
        with open(path, "w") as fh:
            fh.write(json.dumps(meta, indent=2) + "\n")
    except OSError as e:
        raise asb.IoError(f"cannot write sidecar {path}") from e


def open_csv(path: str):
    try:
        return open(path, "w")
    except OSError as e:
        raise asb.IoError(f"cannot write {path}") from e


def probe_config(a) -> asb.ProbeConfig:
    cfg = asb.ProbeConfig.from_env()  # env defaults, flags override
    for name, attr in (("probe_frac", "frac"), ("probe_min_rows", "min_rows"), ("probe_iters", "iters"),
                       ("probe_cap_ms", "cap_ms"), ("probe_topk", "top_k"), ("alpha", "alpha")):
        v = getattr(a, name, None)
        if v is not None:
            setattr(cfg, attr, v)
    return cfg


def probe_json(cfg: asb.ProbeConfig) -> dict:
    return {"frac": cfg.frac, "min_rows": cfg.min_rows, "iters": cfg.iters, "cap_ms": cfg.cap_ms,
            "top_k": cfg.top_k, "alpha": cfg.alpha}


def open_cache(a, cache: asb.ScheduleCache) -> bool:
    """CacheFlags::open (autosage_bench.cpp:117-122): load if present."""
    if not a.cache:
        return False
    if os.path.exists(a.cache):
        cache.load(a.cache)
    return True


def replay_policy(a) -> asb.ReplayPolicy:
    env = asb.ReplayPolicy.from_env()
    return asb.ReplayPolicy(replay_only=env.replay_only or bool(getattr(a, "replay_only", False)),
                            strict=env.strict or bool(getattr(a, "replay_strict", False)))


def load_graph(path: str):
    m = asb.load_csr(path)
    return m, asb.Graph.from_csr(m)


def print_graph_summary(m) -> None:
    """Nearest-rank degree quantiles, rank = ceil(q*n) (src/csr.cpp:97-135), on the host
    (gen needs no GPU)."""
    d = np.sort(m.degrees().astype(np.int64))
    n = d.size

    def q(x):
        return int(d[max(int(np.ceil(x * n)), 1) - 1]) if n else 0
    print(f"nnz={m.nnz}")
    print(f"degree quantiles: p25={q(0.25)} p50={q(0.5)} p75={q(0.75)} p90={q(0.9)} "
          f"p99={q(0.99)} max={int(d[-1]) if n else 0}")


# ---- gen (src/generate.cpp:41-132 shapes; own streams) -------------------------------------
def _csr_from_rows(n_rows: int, n_cols: int, rows) -> asb.CsrMatrix:
    deg = np.array([r.size for r in rows], dtype=np.uint64)
    rowptr = np.zeros(n_rows + 1, dtype=np.uint64)
    rowptr[1:] = np.cumsum(deg)
    colind = (np.concatenate(rows).astype(np.uint32) if rows and rowptr[-1] else np.zeros(0, np.uint32))
    return asb.CsrMatrix(n_rows, n_cols, rowptr, colind, np.ones(colind.size, np.float32))


def _distinct_sorted(rng, n: int, k: int) -> np.ndarray:
    k = min(k, n)
    return np.sort(rng.choice(n, size=k, replace=False))


def gen_er(n: int, p: float, seed: int) -> asb.CsrMatrix:
    rng = np.random.default_rng(seed)
    deg = rng.binomial(n, p, size=n)
    return _csr_from_rows(n, n, [_distinct_sorted(rng, n, int(d)) for d in deg])


def gen_hubskew(n: int, k: int, h: float, seed: int, factor: int) -> asb.CsrMatrix:
    rng = np.random.default_rng(seed)
    hub = rng.random(n) < h
    deg = np.where(hub, k * factor, k)
    return _csr_from_rows(n, n, [_distinct_sorted(rng, n, int(d)) for d in deg])


def gen_hubfixed(n: int, hubs: int, hub_deg: int, other_deg: int, seed: int) -> asb.CsrMatrix:
    rng = np.random.default_rng(seed)
    deg = np.full(n, other_deg)
    deg[:min(hubs, n)] = hub_deg
    return _csr_from_rows(n, n, [_distinct_sorted(rng, n, int(d)) for d in deg])


def run_gen(m, out: str) -> int:
    asb.save_csr(m, out)
    print_graph_summary(m)
    print(f"wrote {out}")
    return EXIT_OK


# ---- bench (autosage_bench.cpp:234-303) ------------------------------------------------------
def run_bench(a) -> int:
    m, g = load_graph(a.graph)
    ds = dataset_name(a.graph)
    dp = asb.DeviceProfile.gpu()
    cfg = probe_config(a)
    cache = asb.ScheduleCache()
    persist = open_cache(a, cache)
    ctx = asb.ScheduleContext(device=dp, cache=cache, replay=replay_policy(a),
                              stream=asb.torch_stream_handle())
    with open_csv(a.out) as csv:
        csv.write("dataset,F,op,choice,baseline_ms,chosen_ms,speedup\n")
        for f in a.f:
            if a.op == "spmm":
                b = seeded_dense(m.n_cols, f, a.seed + f)
                d = asb.decide_spmm(g, b, cfg, ctx)
                base = lambda: asb.spmm_baseline(g, b)  # noqa: E731
                chosen = (lambda: asb.dispatch(d.choice, g, b)) if d.choice else base
            else:
                x = seeded_dense(m.n_rows, f, a.seed + f)
                y = seeded_dense(m.n_cols, f, a.seed + f + 1)
                d = asb.decide_sddmm(g, x, y, cfg, ctx)
                base = lambda: asb.sddmm_baseline(g, x, y)  # noqa: E731
                chosen = (lambda: asb.dispatch(d.choice, g, x, y)) if d.choice else base
            baseline_ms = median_ms(base, a.iters, a.warmups)
            chosen_ms = median_ms(chosen, a.iters, a.warmups)
            b3, c3 = round3(baseline_ms), round3(chosen_ms)
            csv.write(f"{ds},{f},{a.op},{'autosage' if d.choice else 'baseline'},{fmt3(baseline_ms)},"
                      f"{fmt3(chosen_ms)},{fmt3(b3 / c3 if c3 > 0 else 0.0)}\n")
    if persist:
        cache.store(a.cache)
    rp = replay_policy(a)
    write_sidecar(a.out, "bench", dp, {"graph": a.graph, "op": a.op, "f_list": a.f, "iters": a.iters,
                                       "warmups": a.warmups, "probe": probe_json(cfg), "cache": a.cache,
                                       "replay_only": rp.replay_only, "replay_strict": rp.strict,
                                       "seed": a.seed})
    print(f"wrote {a.out}")
    return EXIT_OK


# ---- sweep-split (autosage_bench.cpp:318-363) ------------------------------------------------
def run_sweep_split(a) -> int:
    m, g = load_graph(a.graph)
    ds = dataset_name(a.graph)
    dp = asb.DeviceProfile.gpu()
    b = seeded_dense(m.n_cols, a.f, a.seed)
    ref = asb.spmm_baseline(g, b).cpu().numpy().astype(np.float64)
    baseline_ms = median_ms(lambda: asb.spmm_baseline(g, b), a.iters, a.warmups)
    with open_csv(a.out) as csv:
        csv.write("dataset,F,threshold,baseline_ms,hubsplit_ms,speedup\n")
        for t in a.thresholds:
            v = asb.KernelVariant(asb.SPMM, asb.HUBSPLIT, 64, 4, a.f % 4 == 0, t)
            split = asb.dispatch(v, g, b).output.cpu().numpy()
            # correctness re-check against the baseline before timing (:347-356)
            if np.any(np.abs(split - ref) > 1e-6 + 1e-5 * np.abs(ref)):
                print(f"hubsplit mismatch vs baseline at threshold {t}", file=sys.stderr)
                return EXIT_USAGE
            split_ms = median_ms(lambda: asb.dispatch(v, g, b), a.iters, a.warmups)
            b3, s3 = round3(baseline_ms), round3(split_ms)
            csv.write(f"{ds},{a.f},{t},{fmt3(baseline_ms)},{fmt3(split_ms)},"
                      f"{fmt3(b3 / s3 if s3 > 0 else 0.0)}\n")
    write_sidecar(a.out, "sweep-split", dp, {"graph": a.graph, "f": a.f, "thresholds": a.thresholds,
                                             "iters": a.iters, "warmups": a.warmups, "seed": a.seed})
    print(f"wrote {a.out}")
    return EXIT_OK


# ---- ablate-vec (autosage_bench.cpp:378-428) -------------------------------------------------
def run_ablate_vec(a) -> int:
    m, g = load_graph(a.graph)
    ds = dataset_name(a.graph)
    dp = asb.DeviceProfile.gpu()
    cfg = probe_config(a)
    ctx = asb.ScheduleContext(device=dp, stream=asb.torch_stream_handle())
    op = asb.SPMM if a.op == "spmm" else asb.SDDMM
    with open_csv(a.out) as csv:
        csv.write("dataset,F,op,variant,off_ms,on_ms,speedup\n")
        for f in a.f:
            x = seeded_dense(m.n_rows, f, a.seed + f)
            y = seeded_dense(m.n_cols, f, a.seed + f + 1)
            b = y  # SpMM dense operand, n_cols x f
            d = asb.decide_spmm(g, b, cfg, ctx) if op == asb.SPMM else asb.decide_sddmm(g, x, y, cfg, ctx)
            if d.choice is not None:
                v = d.choice
            elif d.best_index >= 0:
                v = d.candidates[d.best_index].variant
            else:
                v = asb.shortlist(asb.extract_features(m), f, op, dp)[0]
            if f % 4 != 0:
                csv.write(f"{ds},{f},{a.op},{asb.variant_to_string(v)},,,ineligible\n")
                continue
            on = asb.KernelVariant(v.op, v.mapping, v.f_tile, v.rows_per_chunk, True, v.hub_threshold)
            off = asb.KernelVariant(v.op, v.mapping, v.f_tile, v.rows_per_chunk, False, v.hub_threshold)

            def run(kv):
                if op == asb.SPMM:
                    return median_ms(lambda: asb.dispatch(kv, g, b), a.iters, a.warmups)
                return median_ms(lambda: asb.dispatch(kv, g, x, y), a.iters, a.warmups)
            on_ms, off_ms = run(on), run(off)
            on3, off3 = round3(on_ms), round3(off_ms)
            csv.write(f"{ds},{f},{a.op},{asb.variant_to_string(v)},{fmt3(off_ms)},{fmt3(on_ms)},"
                      f"{fmt3(off3 / on3 if on3 > 0 else 0.0)}\n")
    write_sidecar(a.out, "ablate-vec", dp, {"graph": a.graph, "op": a.op, "f_list": a.f, "iters": a.iters,
                                            "warmups": a.warmups, "probe": probe_json(cfg), "seed": a.seed})
    print(f"wrote {a.out}")
    return EXIT_OK


# ---- attention (autosage_bench.cpp:443-524) --------------------------------------------------
def run_attention(a) -> int:
    import torch
    m, g = load_graph(a.graph)
    fv = a.fv or a.f
    ds = dataset_name(a.graph)
    dp = asb.DeviceProfile.gpu()
    cfg = probe_config(a)
    q = seeded_dense(m.n_rows, a.f, a.seed)
    k = seeded_dense(m.n_cols, a.f, a.seed + 1)
    v = seeded_dense(m.n_cols, fv, a.seed + 2)
    cache = asb.ScheduleCache()
    persist = open_cache(a, cache)
    ctx = asb.ScheduleContext(device=dp, cache=cache, stream=asb.torch_stream_handle())
    fused = not a.unfused
    with open_csv(a.out) as csv:
        csv.write("dataset,phase,F,Fv,sddmm_choice,spmm_choice,sddmm_source,spmm_source,"
                  "probe_launches,median_ms\n")

        def emit(phase, run, probes, ms):
            csv.write(f"{ds},{phase},{a.f},{fv},{run.sddmm_decision.choice_string()},"
                      f"{run.spmm_decision.choice_string()},{run.sddmm_decision.source_name},"
                      f"{run.spmm_decision.source_name},{probes},{fmt3(ms)}\n")

        def forward():
            asb.csr_attention_forward(g, q, k, v, cfg, ctx, fused=fused)

        # cold: probes included in the single measured run
        asb.reset_probe_launch_count()
        t0 = time.perf_counter()
        cold = asb.attention_probe_breakdown(g, q, k, v, cfg, ctx, fused=fused)
        torch.cuda.synchronize()
        emit("cold", cold, asb.probe_launch_count(), (time.perf_counter() - t0) * 1e3)
        # warm: cache hits, no probes
        asb.reset_probe_launch_count()
        warm = asb.attention_probe_breakdown(g, q, k, v, cfg, ctx, fused=fused)
        emit("warm", warm, asb.probe_launch_count(), median_ms(forward, a.iters, a.warmups))
        # replay: decisions from the (re-loaded) cache only
        if persist:
            cache.store(a.cache)
            cache.clear()
            cache.load(a.cache)
        ctx.replay = asb.ReplayPolicy(replay_only=True, strict=replay_policy(a).strict)
        asb.reset_probe_launch_count()
        rep = asb.attention_probe_breakdown(g, q, k, v, cfg, ctx, fused=fused)
        emit("replay", rep, asb.probe_launch_count(), median_ms(forward, a.iters, a.warmups))
    if persist:
        cache.store(a.cache)
    write_sidecar(a.out, "attention", dp, {"graph": a.graph, "f": a.f, "fv": fv, "iters": a.iters,
                                           "warmups": a.warmups, "probe": probe_json(cfg), "cache": a.cache,
                                           "seed": a.seed, "fused": fused})
    print(f"wrote {a.out}")
    return EXIT_OK


# ---- replay (autosage_bench.cpp:539-604) -----------------------------------------------------
def run_replay(a) -> int:
    m, g = load_graph(a.graph)
    dp = asb.DeviceProfile.gpu()
    cfg = probe_config(a)
    cache = asb.ScheduleCache()
    cache.load(a.cache)
    strict = a.strict or asb.ReplayPolicy.from_env().strict
    ctx = asb.ScheduleContext(device=dp, cache=cache, replay=asb.ReplayPolicy(True, strict),
                              stream=asb.torch_stream_handle())
    x = seeded_dense(m.n_rows, a.f, a.seed + a.f)
    y = seeded_dense(m.n_cols, a.f, a.seed + a.f + 1)
    b = y
    spmm = a.op == "spmm"
    d = asb.decide_spmm(g, b, cfg, ctx) if spmm else asb.decide_sddmm(g, x, y, cfg, ctx)
    rec = cache.get(d.key)
    if rec is not None:
        if rec.choice != d.choice_string():
            print("replayed decision does not match the cache record", file=sys.stderr)
            return EXIT_USAGE
        print(f"verified: decision matches cache record (t_b={fmt3(rec.t_b)}, t*={fmt3(rec.t_star)}, "
              f"alpha={fmt3(rec.alpha)})")
    else:
        print("cache has no record for this key, served baseline fallback")
    if spmm:
        run = (lambda: asb.dispatch(d.choice, g, b)) if d.choice else (lambda: asb.spmm_baseline(g, b))
    else:
        run = (lambda: asb.dispatch(d.choice, g, x, y)) if d.choice else (lambda: asb.sddmm_baseline(g, x, y))
    ms = median_ms(run, a.iters, a.warmups)
    print(f"key={d.key.to_string()}\nchoice={d.choice_string()}\nsource={d.source_name}\n"
          f"retimed_median_ms={fmt3(ms)}")
    return EXIT_OK


# ---- argument parsing (autosage_bench.cpp:606-731) -------------------------------------------
def _int_list(s: str):
    return [int(t) for t in s.split(",") if t]


def _measure(p, iters=12, warmups=2):
    p.add_argument("--iters", type=int, default=iters, help="Timed iterations per measurement")
    p.add_argument("--warmups", type=int, default=warmups, help="Warm-up iterations per measurement")


def _probe(p):
    p.add_argument("--probe-frac", type=float)
    p.add_argument("--probe-min-rows", type=int)
    p.add_argument("--probe-iters", type=int)
    p.add_argument("--probe-cap-ms", type=float)
    p.add_argument("--probe-topk", type=int)
    p.add_argument("--alpha", type=float, help="Guardrail: accept best iff t* <= alpha*t_b")


def _cache(p):
    p.add_argument("--cache", default=os.environ.get("AUTOSAGE_CACHE", ""),
                   help="Schedule cache file (empty disables persistence)")
    p.add_argument("--replay-only", action="store_true", help="Serve decisions from the cache only, never probe")
    p.add_argument("--replay-strict", action="store_true", help="Make replay misses an error")


def build_parser() -> argparse.ArgumentParser:
    ap = argparse.ArgumentParser(prog="autosage-bench",
                                 description="input-aware scheduling harness for CSR SpMM/SDDMM (B200)")
    sub = ap.add_subparsers(dest="cmd", required=True)

    gen = sub.add_parser("gen", help="Generate a synthetic graph")
    gsub = gen.add_subparsers(dest="kind", required=True)
    er = gsub.add_parser("er", help="Uniform random pattern")
    er.add_argument("--n", type=int, required=True)
    er.add_argument("--p", type=float, required=True)
    hs = gsub.add_parser("hubskew", help="Random hub rows at k*factor degree")
    hs.add_argument("--n", type=int, required=True)
    hs.add_argument("--k", type=int, default=4)
    hs.add_argument("--hub-frac", type=float, default=0.15)
    hs.add_argument("--factor", type=int, default=64)
    hf = gsub.add_parser("hubfixed", help="Fixed hub rows at an exact degree")
    hf.add_argument("--n", type=int, required=True)
    hf.add_argument("--hubs", type=int, default=1)
    hf.add_argument("--hub-deg", type=int, default=5000)
    hf.add_argument("--other-deg", type=int, default=64)
    pl = gsub.add_parser("powerlaw", help="Power-law degrees (device generator, BASELINE configs)")
    pl.add_argument("--n", type=int, required=True)
    pl.add_argument("--nnz", type=int, required=True)
    pl.add_argument("--alpha", type=float, default=2.0)
    pl.add_argument("--dmin", type=int, default=1)
    pl.add_argument("--dmax", type=int, default=0, help="0: n")
    for p in (er, hs, hf, pl):
        p.add_argument("--seed", type=int, default=1)
        p.add_argument("--out", required=True)

    b = sub.add_parser("bench", help="Baseline vs auto-scheduled timing sweep")
    b.add_argument("--graph", required=True)
    b.add_argument("--op", choices=["spmm", "sddmm"], default="spmm")
    b.add_argument("--f", type=_int_list, default=[64], help="Feature widths (comma list)")
    b.add_argument("--seed", type=int, default=1)
    b.add_argument("--out", required=True)
    _measure(b)
    _probe(b)
    _cache(b)

    s = sub.add_parser("sweep-split", help="Baseline vs hub-split threshold sweep")
    s.add_argument("--graph", required=True)
    s.add_argument("--f", type=int, default=128)
    s.add_argument("--thresholds", type=_int_list, default=[64, 256, 1024, 4096])
    s.add_argument("--seed", type=int, default=1)
    s.add_argument("--out", required=True)
    _measure(s)

    v = sub.add_parser("ablate-vec", help="Vec4 on/off ablation (speedup = off/on)")
    v.add_argument("--graph", required=True)
    v.add_argument("--op", choices=["spmm", "sddmm"], default="spmm")
    v.add_argument("--f", type=_int_list, default=[64])
    v.add_argument("--seed", type=int, default=1)
    v.add_argument("--out", required=True)
    _measure(v)
    _probe(v)

    t = sub.add_parser("attention", help="CSR attention pipeline: cold/warm/replay")
    t.add_argument("--graph", required=True)
    t.add_argument("--f", type=int, default=64, help="Q/K feature width")
    t.add_argument("--fv", type=int, default=0, help="V feature width (0: same as --f)")
    t.add_argument("--unfused", action="store_true", help="staged SDDMM -> softmax -> SpMM (default: fused)")
    t.add_argument("--seed", type=int, default=1)
    t.add_argument("--out", required=True)
    _measure(t, 5, 1)
    _probe(t)
    _cache(t)

    r = sub.add_parser("replay", help="Re-run a cached decision without probing")
    r.add_argument("--cache", required=True)
    r.add_argument("--graph", required=True)
    r.add_argument("--op", choices=["spmm", "sddmm"], default="spmm")
    r.add_argument("--f", type=int, default=64)
    r.add_argument("--strict", action="store_true", help="Treat a replay miss as an error")
    r.add_argument("--seed", type=int, default=1)
    _measure(r)
    _probe(r)
    return ap


def dispatch_command(a) -> int:
    if a.cmd == "gen":
        if a.kind == "er":
            return run_gen(gen_er(a.n, a.p, a.seed), a.out)
        if a.kind == "hubskew":
            return run_gen(gen_hubskew(a.n, a.k, a.hub_frac, a.seed, a.factor), a.out)
        if a.kind == "hubfixed":
            return run_gen(gen_hubfixed(a.n, a.hubs, a.hub_deg, a.other_deg, a.seed), a.out)
        return run_gen(asb.gen_powerlaw(a.n, a.n, a.nnz, a.alpha, a.dmin, a.dmax or a.n, a.seed), a.out)
    return {"bench": run_bench, "sweep-split": run_sweep_split, "ablate-vec": run_ablate_vec,
            "attention": run_attention, "replay": run_replay}[a.cmd](a)


def main(argv=None) -> int:
    ap = build_parser()
    try:
        a = ap.parse_args(argv)
    except SystemExit as e:  # argparse: --help exits 0, parse errors 2 -> usage (1)
        return EXIT_OK if e.code == 0 else EXIT_USAGE
    try:
        return dispatch_command(a)
    except asb.ReplayMiss as e:  # autosage_bench.cpp:733-750
        print(f"error: {e}", file=sys.stderr)
        return EXIT_REPLAY_MISS
    except (asb.IoError, asb.CacheError, OSError) as e:
        print(f"error: {e}", file=sys.stderr)
        return EXIT_IO
    except Exception as e:  # noqa: BLE001
        print(f"error: {e}", file=sys.stderr)
        return EXIT_USAGE


if __name__ == "__main__":
    sys.exit(main())
