#!/usr/bin/env python3
"""AutoSAGE-B200 benchmark (driver contract).

One step = one pass of the hot path over the configured synthetic graph:
the scheduler's chosen SpMM (C = A*B) and SDDMM (out = <X_i, Y_j> on A's
pattern) through the library's input-aware entry points (as_spmm_auto /
as_sddmm_auto, decisions cached after one cold probe), inputs resident in
HBM.  `value` = gather-model bytes of both ops (the reference's
own cost formulas, proj/src/cost.cpp:21-27) over all ranks / max-rank time.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config reddit]
  python bench.py --impl reference ...   # reference CPU library, host cores

Multi-GPU (torchrun): rows are nnz-balanced across ranks (as_partition_rows);
each step all-gathers the dense B/Y row shards over NCCL, then runs the
local SpMM/SDDMM on the rank's row range ("strong" scaling).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

# name -> (n_rows, nnz, alpha, d_min, d_max, F); degree shapes in DESIGN.md
CONFIGS = {
    "c1": (100_000, 1_600_000, 2.5, 6, 2000, 64),
    "reddit": (232_965, 114_615_892, 2.2, 100, 21_657, 64),
    "products": (2_449_029, 123_718_280, 2.0, 8, 17_481, 100),
    # diagnostics: Reddit volume with the degree tail capped
    "reddit_cap2k": (232_965, 114_615_892, 2.2, 100, 2048, 64),
}
L2_FLUSH_BYTES = 256 << 20
PEAK_FALLBACK_GBS = 6650.0


def gather_bytes(op: str, n_rows: int, nnz: int, f: int) -> float:
    """proj/src/cost.cpp:21-27 (the reference cost model's traffic)."""
    if op == "spmm":
        return 8.0 * nnz + 4.0 * nnz * f + 4.0 * n_rows * f + 8.0 * (n_rows + 1)
    return 8.0 * nnz + 8.0 * nnz * f + 4.0 * nnz


def measured_peak():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as fh:
            return float(json.load(fh)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return PEAK_FALLBACK_GBS, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append((time.time(), line.strip()))

    def window(self, t0, t1):
        """Keep samples inside [t0, t1] (plus the nearest one on each side
        when the window is shorter than the sampling period)."""
        inside = [x for x in self.lines if t0 <= x[0] <= t1]
        before = [x for x in self.lines if x[0] < t0][-1:]
        after = [x for x in self.lines if x[0] > t1][:1]
        self.lines = inside if len(inside) >= 3 else before + inside + after

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for _, ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) != 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for n, v in zip(names, parts[2:]):
                if v.lower() == "active":
                    reasons.add(n)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx), "reasons": sorted(reasons),
                "samples": len(sm)}


def make_graph(cfg_name: str, seed: int):
    import paper_2511_17594_b200 as asb
    n, nnz, alpha, dmin, dmax, f = CONFIGS[cfg_name]
    m = asb.gen_powerlaw(n, n, nnz, alpha, dmin, dmax, seed)
    return m, f


def host_row_sample(m, step: int):
    """Every `step`-th row (a systematic sample) as a host CSR."""
    import paper_2511_17594_b200 as asb
    rows = np.arange(0, m.n_rows, step)
    deg = (m.rowptr[rows + 1] - m.rowptr[rows]).astype(np.int64)
    rp = np.zeros(rows.size + 1, dtype=np.uint64)
    rp[1:] = np.cumsum(deg)
    idx = np.concatenate([np.arange(m.rowptr[r], m.rowptr[r + 1], dtype=np.int64) for r in rows])
    return asb.CsrMatrix(rows.size, m.n_cols, rp, m.colind[idx],
                         None if m.val is None else m.val[idx]), rows


# ---------------------------------------------------------------------------
# reference CPU arm
# ---------------------------------------------------------------------------
def cpu_reference_run(m, f, seed, steps, warmup, sample_step):
    """Reference library (oracle/_ref, else the C port) on the host cores:
    decide once with the reference scheduler, then time dispatch(choice)
    SpMM + SDDMM per step on a systematic row sample of the workload."""
    import oracle
    import paper_2511_17594_b200 as asb
    sm, rows = host_row_sample(m, sample_step)
    b = asb.fill_uniform(m.n_cols * f, seed + f, (m.n_cols, f))
    x = asb.fill_uniform(m.n_rows * f, seed + f, (m.n_rows, f))[rows]
    y = asb.fill_uniform(m.n_cols * f, seed + f + 1, (m.n_cols, f))
    total = gather_bytes("spmm", sm.n_rows, sm.nnz, f) + gather_bytes("sddmm", sm.n_rows, sm.nnz, f)
    if oracle.ref_available():
        kind, cores = "reference", oracle.ref_default_workers()
        rg, rb, rx, ry = oracle.RefGraph(sm), oracle.RefDense(b), oracle.RefDense(x), oracle.RefDense(y)
        spmm_choice, _ = oracle.ref_decide(rg, None, rb, 0)
        sddmm_choice, _ = oracle.ref_decide(rg, rx, ry, 1)
        out = np.empty((sm.n_rows, f), np.float32)

        def step():
            if spmm_choice == "baseline":
                oracle.ref_spmm_baseline(rg, rb)
            else:
                oracle.ref_spmm_dispatch(spmm_choice, rg, rb, 0, out)
            if sddmm_choice == "baseline":
                oracle.ref_sddmm_baseline(rg, rx, ry)
            else:
                oracle.ref_sddmm_dispatch(sddmm_choice, rg, rx, ry, 0)
        choices = {"spmm": spmm_choice, "sddmm": sddmm_choice}
    else:
        kind, cores = "port", 1
        choices = {"spmm": "baseline", "sddmm": "baseline"}

        def step():
            oracle.spmm_baseline(sm, b)
            oracle.sddmm(sm, x, y)
    for _ in range(warmup):
        step()
    t0 = time.perf_counter()
    for _ in range(steps):
        step()
    dt = time.perf_counter() - t0
    gbs = total * steps / dt / 1e9
    sample = (f"every {sample_step}th row of the workload ({sm.n_rows} rows, {sm.nnz} nnz, F={f}); "
              f"SpMM {choices['spmm']} + SDDMM {choices['sddmm']}; {steps} timed steps")
    return {"value": gbs, "unit": "GB/s", "cores": int(cores), "kind": kind, "sample": sample,
            "ms_per_step": dt / steps * 1e3}


def run_reference_arm(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    m, f = make_graph(args.config, args.seed)
    steps, warmup = args.steps, args.warmup
    cpu = cpu_reference_run(m, f, args.seed, steps, warmup, args.cpu_sample_step)
    line = {
        "impl": "reference", "metric": metric_name(args.config, f), "value": cpu["value"],
        "unit": "GB/s", "n_gpus": args.gpus, "steps": steps, "warmup": warmup,
        "ms_per_step": cpu["ms_per_step"], "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": workload_name(args.config, f), "n_rows": m.n_rows, "nnz": m.nnz,
                   "F": f, "sample": cpu["sample"]},
        "cpu_baseline": {k: cpu[k] for k in ("value", "unit", "cores", "kind", "sample")},
        "e2e": {"value": cpu["value"], "unit": "GB/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def metric_name(cfg, f):
    return f"SpMM+SDDMM gather-model GB/s ({cfg}-shaped CSR, F={f})"


def workload_name(cfg, f):
    n, nnz = CONFIGS[cfg][0], CONFIGS[cfg][1]
    return f"{cfg}-shaped power-law CSR N={n} nnz={nnz}, SpMM + SDDMM at F={f}"


# ---------------------------------------------------------------------------
# B200 arm
# ---------------------------------------------------------------------------
def run_ours(args):
    import torch
    import paper_2511_17594_b200 as asb
    import ctypes as C
    from paper_2511_17594_b200 import _capi

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)
    stream = torch.cuda.current_stream(dev)

    m, f = make_graph(args.config, args.seed)
    if args.f:
        f = args.f
    n_rows, nnz = m.n_rows, m.nnz
    from paper_2511_17594_b200.dist import RowSharding
    sh = RowSharding(m.rowptr, world, rank)  # nnz-balanced contiguous row ranges
    r0, r1 = sh.r0, sh.r1
    # N>1: this rank's rows, columns remapped into the padded all-gather layout
    # (dist.py), so the kernels gather straight from the NCCL buffer
    g = asb.Graph.from_csr(m if world == 1 else sh.shard_graph_host(m), device=local)
    # dense operands (reference bench seeds: B seed+F, X seed+F, Y seed+F+1)
    b_host = asb.fill_uniform(m.n_cols * f, args.seed + f, (m.n_cols, f))
    x_host = asb.fill_uniform(n_rows * f, args.seed + f, (n_rows, f))
    y_host = asb.fill_uniform(m.n_cols * f, args.seed + f + 1, (m.n_cols, f))
    # square graph: rank r owns the B/Y rows of its own node range
    b_full = torch.from_numpy(b_host).to(dev)
    y_full = torch.from_numpy(y_host).to(dev)
    x_loc = torch.from_numpy(x_host[r0:r1]).to(dev)
    if world > 1:
        # own rows as the all-gather input in place (padded to the largest shard)
        b_loc = torch.zeros((sh.shard, f), dtype=torch.float32, device=dev)
        y_loc = torch.zeros((sh.shard, f), dtype=torch.float32, device=dev)
        b_loc[: r1 - r0] = b_full[r0:r1]
        y_loc[: r1 - r0] = y_full[r0:r1]
        pad_b = torch.zeros((sh.padded_rows, f), dtype=torch.float32, device=dev)
        pad_y = torch.zeros((sh.padded_rows, f), dtype=torch.float32, device=dev)
        del b_full, y_full
        # the e2e leg feeds the same layout from the host
        b_host_e2e = np.zeros((sh.padded_rows, f), dtype=np.float32)
        y_host_e2e = np.zeros((sh.padded_rows, f), dtype=np.float32)
        b_host_e2e[sh.perm] = b_host
        y_host_e2e[sh.perm] = y_host
    else:
        b_host_e2e, y_host_e2e = b_host, y_host
    c = torch.empty((r1 - r0, f), dtype=torch.float32, device=dev)
    sv = torch.empty(max(g.nnz, 1), dtype=torch.float32, device=dev)
    flush = torch.empty(L2_FLUSH_BYTES // 4, dtype=torch.float32, device=dev)

    cache = asb.ScheduleCache()
    if args.cache and os.path.exists(args.cache):
        cache.load(args.cache)  # deterministic replay of an earlier run's decisions
    ctx = asb.ScheduleContext(cache=cache, stream=asb.torch_stream_handle(dev),
                              replay=asb.ReplayPolicy(replay_only=args.replay_only,
                                                      strict=args.replay_only))
    cfg = asb.ProbeConfig.from_env()
    cctx, keep = ctx.to_c()
    ccfg = cfg.to_c()
    d_spmm, d_sddmm = _capi.as_decision(), _capi.as_decision()
    lib = _capi.lib

    def P(t):
        return C.c_void_p(t.data_ptr())

    def gather_b():
        """B for the SpMM; starts Y's all-gather on NCCL's stream so it runs
        under the SpMM (returned handle: wait before the SDDMM)."""
        if world == 1:
            return b_full, None
        sh.allgather_padded(b_loc, pad_b)
        return pad_b, sh.allgather_padded(y_loc, pad_y, async_op=True)

    def y_operand(hy):
        if world == 1:
            return y_full
        hy.wait()
        return pad_y

    def spmm(bm):
        asb._check(lib.as_spmm_auto(C.byref(cctx), C.byref(ccfg), g.handle, P(bm), bm.shape[0], f,
                                    P(c), C.byref(d_spmm)))

    def sddmm(ym):
        asb._check(lib.as_sddmm_auto(C.byref(cctx), C.byref(ccfg), g.handle, P(x_loc), r1 - r0,
                                     P(ym), ym.shape[0], f, P(sv), C.byref(d_sddmm)))

    # cold decisions (probes) -- outside the timed region, reported separately
    t0 = time.perf_counter()
    bm, hy = gather_b()
    spmm(bm)
    sddmm(y_operand(hy))
    torch.cuda.synchronize(dev)
    cold_ms = (time.perf_counter() - t0) * 1e3
    dec_spmm = asb.ScheduleDecision.from_c(d_spmm)
    dec_sddmm = asb.ScheduleDecision.from_c(d_sddmm)
    if args.cache and rank == 0 and not args.replay_only:
        cache.store(args.cache)

    ev = [[torch.cuda.Event(enable_timing=True) for _ in range(4)] for _ in range(args.steps)]

    def step(i=None):
        flush.zero_()  # L2 flush between steps (untimed)
        e = ev[i] if i is not None else None
        if e:
            e[0].record(stream)
        bm, hy = gather_b()
        if e:
            e[1].record(stream)
        spmm(bm)
        if e:
            e[2].record(stream)
        sddmm(y_operand(hy))  # Y's all-gather overlapped the SpMM
        if e:
            e[3].record(stream)

    with ClockSampler(local) as clocks:
        for _ in range(args.warmup):
            step()
        torch.cuda.synchronize(dev)
        if dist:
            dist.barrier()
        launches0 = asb.kernel_launch_count()
        tw0 = time.time()
        for i in range(args.steps):
            step(i)
        torch.cuda.synchronize(dev)
        tw1 = time.time()
        if dist:
            dist.barrier()
        time.sleep(0.25)  # let the sampler report the tail of the window
    clocks.window(tw0, tw1)
    launches = asb.kernel_launch_count() - launches0
    t_gather = sum(e[0].elapsed_time(e[1]) for e in ev)
    t_spmm = sum(e[1].elapsed_time(e[2]) for e in ev)
    t_sddmm = sum(e[2].elapsed_time(e[3]) for e in ev)
    total = t_gather + t_spmm + t_sddmm
    if dist:
        tt = torch.tensor([total, t_gather, t_spmm, t_sddmm], dtype=torch.float64, device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        total, t_gather, t_spmm, t_sddmm = tt.tolist()
    K = args.steps
    bytes_spmm = gather_bytes("spmm", n_rows, nnz, f)
    bytes_sddmm = gather_bytes("sddmm", n_rows, nnz, f)
    value = (bytes_spmm + bytes_sddmm) * K / (total * 1e-3) / 1e9
    peak, peak_src = measured_peak()

    # roofline of the dominant op (its algorithmic bytes per launch on this rank)
    local_nnz = g.nnz
    lb_spmm = gather_bytes("spmm", r1 - r0, local_nnz, f)
    lb_sddmm = gather_bytes("sddmm", r1 - r0, local_nnz, f)
    dom = "sddmm" if t_sddmm >= t_spmm else "spmm"
    dom_ms = (t_sddmm if dom == "sddmm" else t_spmm) / K
    dom_bytes = lb_sddmm if dom == "sddmm" else lb_spmm
    achieved = dom_bytes / (dom_ms * 1e-3) / 1e9
    traffic = None
    tp = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tp):
        try:
            with open(tp) as fh:
                traffic = json.load(fh).get(f"{args.config}:F={f}:{dom}")
        except Exception:
            traffic = None

    # e2e through the reference-facing host-buffer entry points
    e2e = None
    if not args.no_e2e:
        # every rank: full B/Y and its own X rows in, its own C rows and SDDMM
        # values out, through the host-buffer API; time = max over ranks
        e2e = run_e2e(args, g, f, r1 - r0, b_host_e2e, x_host[r0:r1], y_host_e2e, dec_spmm, dec_sddmm,
                      bytes_spmm + bytes_sddmm, dist)

    cpu = None
    if world == 1 and rank == 0 and not args.no_cpu:
        cpu = cpu_reference_run(m, f, args.seed, 2, 1, args.cpu_sample_step)
        cpu.pop("ms_per_step", None)

    if rank == 0:
        clk = clocks.summary()
        line = {
            "metric": metric_name(args.config, f), "value": value, "unit": "GB/s",
            "n_gpus": world, "steps": K, "warmup": args.warmup, "ms_per_step": total / K,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic",
            "config": {"workload": workload_name(args.config, f), "n_rows": n_rows, "nnz": nnz,
                       "F": f, "parallelism": f"row-sharded x{world}" if world > 1 else "1 GPU",
                       "l2": "flushed between steps (256 MiB write, untimed)",
                       "exchange": ("none (1 GPU)" if world == 1 else
                                    "NCCL all-gather of B row shards before the SpMM; Y's all-gather on "
                                    "NCCL's stream under the SpMM; kernels read the padded buffers in place"),
                       "spmm_choice": dec_spmm.choice_string(),
                       "sddmm_choice": dec_sddmm.choice_string(),
                       "decision_source": {"spmm": dec_spmm.source_name,
                                           "sddmm": dec_sddmm.source_name},
                       "probe": dataclasses_asdict(cfg)},
            "ms_per_op": {"spmm": t_spmm / K, "sddmm": t_sddmm / K, "allgather": t_gather / K},
            # 2*nnz*F flops per op (proj/src/cost.cpp:28), whole job
            "gflops_per_s": {"spmm": 2.0 * nnz * f / (t_spmm / K * 1e-3) / 1e9,
                             "sddmm": 2.0 * nnz * f / (t_sddmm / K * 1e-3) / 1e9,
                             "step": 4.0 * nnz * f / (total / K * 1e-3) / 1e9},
            "pct_of_8TBs": value / 8000.0 * 100.0,
            "decide_cold_ms": cold_ms,
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic, "kernel": dom,
                         "bytes_model": "gather model, proj/src/cost.cpp:21-27", "peak_source": peak_src,
                         # measured DRAM bytes over the same time: the gathers hit L2,
                         # so the op is bound on chip, not by HBM
                         "dram_gbs": (traffic / (dom_ms * 1e-3) / 1e9) if traffic else None,
                         "dram_frac": (traffic / (dom_ms * 1e-3) / 1e9 / peak) if traffic else None,
                         "binding_resource": {"sddmm": "shared-memory datapath (Y staging + X broadcast)",
                                              "spmm": "L2 gather latency (long scoreboard)"}[dom]},
            "gpu_launches": int(launches),
            "clocks": clk,
        }
        if e2e:
            line["e2e"] = e2e
        if cpu:
            line["cpu_baseline"] = cpu
        print(json.dumps(line), flush=True)
    del keep
    if dist:
        dist.destroy_process_group()


def dataclasses_asdict(cfg):
    import dataclasses
    return dataclasses.asdict(cfg)


def run_e2e(args, g, f, n_rows, b_host, x_host, y_host, dec_spmm, dec_sddmm, step_bytes, dist=None):
    """Same step through the host-buffer C-ABI: as_spmm_host_async +
    as_sddmm_host_async + as_graph_synchronize, pinned host buffers.  The H2D
    of B/X/Y and the D2H of C and of the SDDMM values are inside the timed
    region; the library overlaps them with the kernels (copy-in / compute /
    copy-out streams, SDDMM values returned in slices)."""
    import torch
    import ctypes as C
    import paper_2511_17594_b200 as asb
    from paper_2511_17594_b200 import _capi
    lib = _capi.lib
    pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory()  # noqa: E731
    b, x, y = pin(b_host), pin(x_host), pin(y_host)
    c = torch.empty((n_rows, f), dtype=torch.float32).pin_memory()
    sv = torch.empty(max(g.nnz, 1), dtype=torch.float32).pin_memory()
    vs = dec_spmm.choice.to_c() if dec_spmm.choice else None
    vd = dec_sddmm.choice.to_c() if dec_sddmm.choice else None
    res = _capi.as_kernel_result()

    def step():
        # SDDMM first: its values are most of the D2H bytes, so their copies
        # should start as early as possible
        asb._check(lib.as_sddmm_host_async(C.byref(vd) if vd else None, g.handle,
                                           C.c_void_p(x.data_ptr()), x.shape[0],
                                           C.c_void_p(y.data_ptr()), y.shape[0], f,
                                           C.c_void_p(sv.data_ptr()), C.byref(res)))
        asb._check(lib.as_spmm_host_async(C.byref(vs) if vs else None, g.handle,
                                          C.c_void_p(b.data_ptr()), b.shape[0], f,
                                          C.c_void_p(c.data_ptr()), C.byref(res)))
        asb._check(lib.as_graph_synchronize(g.handle))
    step()
    k = max(3, min(args.steps, 10))
    times = []
    for _ in range(k):
        if dist:
            dist.barrier()
        t0 = time.perf_counter()
        step()
        times.append(time.perf_counter() - t0)
    if dist:  # per step, the slowest rank
        tt = torch.tensor(times, dtype=torch.float64, device="cuda")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        times = tt.tolist()
    dt = statistics.median(times)
    h2d = (b_host.nbytes + x_host.nbytes + y_host.nbytes)
    d2h_local = n_rows * f * 4 + g.nnz * 4
    d2h = d2h_local
    if dist:  # whole-job bytes moved
        bt = torch.tensor([h2d, d2h], dtype=torch.float64, device="cuda")
        dist.all_reduce(bt)
        h2d, d2h = int(bt[0].item()), int(bt[1].item())
    # the link alone: this rank's D2H bytes copied device -> pinned host with
    # no kernels (what the pipeline cannot go below)
    dev_buf = torch.empty(d2h_local // 4, dtype=torch.float32, device="cuda")
    host_buf = torch.empty(d2h_local // 4, dtype=torch.float32).pin_memory()
    copy_ms = []
    for _ in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        host_buf.copy_(dev_buf, non_blocking=True)
        e1.record()
        e1.synchronize()
        copy_ms.append(e0.elapsed_time(e1))
    d2h_floor_ms = min(copy_ms)
    del dev_buf, host_buf
    return {"value": step_bytes / dt / 1e9, "unit": "GB/s", "h2d_bytes_per_step": int(h2d),
            "d2h_bytes_per_step": int(d2h), "ms_per_step": dt * 1e3, "steps": k,
            "d2h_copy_only_ms": d2h_floor_ms, "d2h_gbs": d2h_local / (d2h_floor_ms * 1e-3) / 1e9,
            "timing": "host wall clock per step (median), synchronize at the end of each step",
            "api": "as_sddmm_host_async + as_spmm_host_async + as_graph_synchronize "
                   "(decided variants), pinned host buffers"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="reddit", choices=sorted(CONFIGS))
    ap.add_argument("--f", type=int, default=0, help="override feature width")
    ap.add_argument("--seed", type=int, default=1)
    ap.add_argument("--cpu-sample-step", type=int, default=8)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--cache", default="", help="schedule cache file: load if present, store after decide")
    ap.add_argument("--replay-only", action="store_true",
                    help="decisions must come from --cache (strict replay, no probes)")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        run_reference_arm(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
