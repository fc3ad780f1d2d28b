#!/usr/bin/env python3
"""Measurement sweep over the BASELINE.json configs on one GPU.

  python tools/sweep.py [--cases c1,c2,c3,c4,c5] [--out gpurun_out/sweep.json]

c1  SpMM+SDDMM on the 100k-row power-law graph, F=64 (+ reference CPU library on
    the same graph, all host cores)
c2  Reddit-shape SpMM + SDDMM at F = 32 / 64 / 128 / 256
c3  Products-shape SpMM F=100: per-rank compute of the nnz-balanced row shards
    for g = 1, 2, 4, 8 (each shard timed alone on this GPU with the full B
    resident; the all-gather is not included -- one GPU here)
c4  skew stressor: Zipf exponents 1.5 / 2.0 / 2.5 / 3.0, hubs up to 1M nnz,
    F = 16 / 64 / 128: decision, guardrail (chosen vs baseline on the full
    graph) and cache replay (a fresh context replaying the stored decisions)
c5  CSR attention on Reddit-shape, 8 heads x F=64: fused vs unfused per head
bwd backward pieces on Reddit-shape F=64: transpose build, dB = A^T dC, dval = SDDMM(dC, B),
    row-softmax gradient, torch autograd of spmm_csr / csr_attention
bf16 SpMM with a bf16 B (as_spmm_bf16) beside f32 on Reddit F=32/64/128 and Products F=100

Every GPU time is CUDA events on the launching stream around `reps` launches
(median per launch), decisions made once before timing.  Bytes are the
reference gather model (proj/src/cost.cpp:21-27).
"""
import argparse
import ctypes as C
import json
import os
import statistics
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2511_17594_b200 as asb  # noqa: E402
from paper_2511_17594_b200 import _capi  # noqa: E402

lib = _capi.lib
PEAK, _ = bench.measured_peak()


def P(t):
    return C.c_void_p(t.data_ptr())


_FLUSH = None


def ev_time(fn, reps=5, warm=2):
    """Median per-call GPU ms of fn(): CUDA events around each call, calls
    queued back to back with a 256 MB L2-flush write between them (outside
    the events; it also gives the host time to enqueue the next call), one
    synchronize at the end -- the device time of a call, as bench.py times
    its steps (round-1/2 sweeps up to r02l synchronized after every call, so
    their small-graph times include the host enqueue)."""
    global _FLUSH
    if _FLUSH is None:
        _FLUSH = torch.empty(64 << 20, dtype=torch.float32, device="cuda")
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    evs = []
    for _ in range(reps):
        _FLUSH.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        evs.append((e0, e1))
    torch.cuda.synchronize()
    return statistics.median(e0.elapsed_time(e1) for e0, e1 in evs)


class Ops:
    """Device-pointer calls through the C-ABI on torch's current stream."""

    def __init__(self, g, f):
        self.g, self.f = g, f
        self.stream = C.c_void_p(asb.torch_stream_handle())

    def spmm(self, v, b, c):
        cv = v.to_c() if v else None
        asb._check(lib.as_spmm(C.byref(cv) if cv else None, self.g.handle, P(b), b.shape[0], self.f,
                               P(c), self.stream, None))

    def sddmm(self, v, x, y, out):
        cv = v.to_c() if v else None
        asb._check(lib.as_sddmm(C.byref(cv) if cv else None, self.g.handle, P(x), x.shape[0], P(y),
                                y.shape[0], self.f, P(out), self.stream, None))


def gbs(op, n, nnz, f, ms):
    return bench.gather_bytes(op, n, nnz, f) / (ms * 1e-3) / 1e9


def decide(op, g, f, dev_in, ctx, cfg):
    if op == "spmm":
        return asb.decide_spmm(g, dev_in[0], cfg, ctx)
    return asb.decide_sddmm(g, dev_in[0], dev_in[1], cfg, ctx)


def run_graph(m, f, ops=("spmm", "sddmm"), reps=5, seed=1, with_baseline=True, cache=None):
    g = asb.Graph.from_csr(m)
    dev = torch.device("cuda")
    b = torch.from_numpy(asb.fill_uniform(m.n_cols * f, seed + f, (m.n_cols, f))).to(dev)
    x = torch.from_numpy(asb.fill_uniform(m.n_rows * f, seed + f, (m.n_rows, f))).to(dev)
    y = torch.from_numpy(asb.fill_uniform(m.n_cols * f, seed + f + 1, (m.n_cols, f))).to(dev)
    c = torch.empty((m.n_rows, f), dtype=torch.float32, device=dev)
    sv = torch.empty(max(m.nnz, 1), dtype=torch.float32, device=dev)
    cache = cache or asb.ScheduleCache()
    ctx = asb.ScheduleContext(cache=cache, stream=asb.torch_stream_handle())
    cfg = asb.ProbeConfig.from_env()
    o = Ops(g, f)
    out = {}
    for op in ops:
        t0 = time.perf_counter()
        d = decide(op, g, f, (b,) if op == "spmm" else (x, y), ctx, cfg)
        cold = (time.perf_counter() - t0) * 1e3
        v = d.choice
        if op == "spmm":
            t = ev_time(lambda: o.spmm(v, b, c), reps)
            tb = ev_time(lambda: o.spmm(None, b, c), max(2, reps // 2)) if with_baseline else None
        else:
            t = ev_time(lambda: o.sddmm(v, x, y, sv), reps)
            tb = ev_time(lambda: o.sddmm(None, x, y, sv), max(2, reps // 2)) if with_baseline else None
        out[op] = {"choice": d.choice_string(), "source": d.source_name, "ms": t,
                   "gbs": gbs(op, m.n_rows, m.nnz, f, t), "frac_hbm": gbs(op, m.n_rows, m.nnz, f, t) / PEAK,
                   "baseline_ms": tb, "decide_cold_ms": cold,
                   "probe": {"t_b": d.baseline_ms, "t_star": d.t_star, "sample_rows": d.sample_rows,
                             "candidates": [(asb.variant_to_string(ct.variant), ct.median_ms)
                                            for ct in d.candidates]}}
    g.close()
    return out, cache


def case_c1(res):
    m, f = bench.make_graph("c1", 1)
    r, _ = run_graph(m, f, reps=20)
    cpu, _ = bench.cpu_reference_run(m, f, 1, 12, 2, "c1")
    cpu = {k: v for k, v in cpu.items() if k != "choices"}
    res["c1"] = {"graph": {"n": m.n_rows, "nnz": m.nnz, "F": f}, "gpu": r, "cpu_reference": cpu}


def cusparse_times(m, f, reps=5):
    """cuSPARSE through torch (fp32 accumulation -- a speed reference only, not
    the reference numerics): CSR SpMM (torch.sparse.mm) and CSR SDDMM
    (torch.sparse.sampled_addmm)."""
    dev = torch.device("cuda")
    rp = torch.from_numpy(m.rowptr.astype(np.int64)).to(dev)
    ci = torch.from_numpy(m.colind.astype(np.int64)).to(dev)
    val = torch.from_numpy(m.val if m.val is not None else np.ones(m.nnz, np.float32)).to(dev)
    a = torch.sparse_csr_tensor(rp, ci, val, (m.n_rows, m.n_cols))
    b = torch.from_numpy(asb.fill_uniform(m.n_cols * f, 1 + f, (m.n_cols, f))).to(dev)
    x = torch.from_numpy(asb.fill_uniform(m.n_rows * f, 1 + f, (m.n_rows, f))).to(dev)
    out = {}
    try:
        out["spmm_ms"] = ev_time(lambda: torch.sparse.mm(a, b), reps)
    except Exception as e:  # pragma: no cover
        out["spmm_error"] = str(e)[:200]
    try:
        pat = torch.sparse_csr_tensor(rp, ci, torch.ones_like(val), (m.n_rows, m.n_cols))
        yt = b.t().contiguous()
        out["sddmm_ms"] = ev_time(lambda: torch.sparse.sampled_addmm(pat, x, yt, beta=0.0, alpha=1.0), reps)
    except Exception as e:  # pragma: no cover
        out["sddmm_error"] = str(e)[:200]
    return out


def case_c2(res):
    m, _ = bench.make_graph("reddit", 1)
    res["c2"] = {"graph": {"n": m.n_rows, "nnz": m.nnz}, "by_F": {}, "cusparse": {}}
    for f in (32, 64, 128, 256):
        r, _ = run_graph(m, f, reps=5, with_baseline=(f <= 64))
        res["c2"]["by_F"][str(f)] = r
        res["c2"]["cusparse"][str(f)] = cusparse_times(m, f)


def case_c3(res):
    m, f = bench.make_graph("products", 1)
    from paper_2511_17594_b200.dist import RowSharding
    g_full = asb.Graph.from_csr(m)
    dev = torch.device("cuda")
    b = torch.from_numpy(asb.fill_uniform(m.n_cols * f, 1 + f, (m.n_cols, f))).to(dev)
    ctx = asb.ScheduleContext(cache=asb.ScheduleCache(), stream=asb.torch_stream_handle())
    cfg = asb.ProbeConfig.from_env()
    d = asb.decide_spmm(g_full, b, cfg, ctx)
    v = d.choice
    out = {"graph": {"n": m.n_rows, "nnz": m.nnz, "F": f}, "choice": d.choice_string(), "by_g": {}}
    for world in (1, 2, 4, 8):
        per_rank = []
        for rank in range(world):
            sh = RowSharding(m.rowptr, world, rank)
            gs = g_full if world == 1 else g_full.row_range(sh.r0, sh.r1)
            c = torch.empty((sh.r1 - sh.r0, f), dtype=torch.float32, device=dev)
            o = Ops(gs, f)
            per_rank.append(ev_time(lambda: o.spmm(v, b, c), 5))
            if world > 1:
                gs.close()
        worst = max(per_rank)
        out["by_g"][str(world)] = {"per_rank_ms": per_rank, "max_rank_ms": worst,
                                   "gbs_total": gbs("spmm", m.n_rows, m.nnz, f, worst),
                                   "allgather_bytes_per_rank": int((world - 1) * (m.n_cols // world) * f * 4)}
    base = out["by_g"]["1"]["max_rank_ms"]
    for k, e in out["by_g"].items():
        e["compute_speedup"] = base / e["max_rank_ms"]
    g_full.close()
    res["c3"] = out


with_hubs = bench.with_hubs


def case_c4(res):
    out = []
    n = 1_100_000
    for alpha in (1.5, 2.0, 2.5, 3.0):
        m = with_hubs(asb.gen_powerlaw(n, n, 24_000_000, alpha, 4, 1_000_000, 7),
                      [1_000_000, 250_000, 60_000], 11)
        deg = np.diff(m.rowptr.astype(np.int64))
        for f in (16, 64, 128):
            r, cache = run_graph(m, f, ops=("spmm",), reps=3)
            # replay: a fresh context that must reproduce the stored decision
            fd, path = tempfile.mkstemp(suffix=".cache")
            os.close(fd)
            cache.store(path)
            c2 = asb.ScheduleCache()
            c2.load(path)
            os.unlink(path)
            r2, _ = run_graph(m, f, ops=("spmm",), reps=2, with_baseline=False, cache=c2)
            e = r["spmm"]
            out.append({"alpha": alpha, "F": f, "n": m.n_rows, "nnz": m.nnz, "deg_max": int(deg.max()),
                        "choice": e["choice"], "ms": e["ms"], "baseline_ms": e["baseline_ms"],
                        "guardrail_ok": e["ms"] <= e["baseline_ms"] * 1.02,
                        "gbs": e["gbs"], "probe": e["probe"],
                        "replay_source": r2["spmm"]["source"],
                        "replay_same_choice": r2["spmm"]["choice"] == e["choice"]})
        del m
    res["c4"] = out


def case_c5(res):
    m, _ = bench.make_graph("reddit", 1)
    f = 64
    g = asb.Graph.from_csr(m)
    dev = torch.device("cuda")
    cache = asb.ScheduleCache()
    ctx = asb.ScheduleContext(cache=cache, stream=asb.torch_stream_handle())
    cfg = asb.ProbeConfig.from_env()
    cctx, keep = ctx.to_c()
    ccfg = cfg.to_c()
    out_t = torch.empty((m.n_rows, f), dtype=torch.float32, device=dev)
    sd, pd = _capi.as_decision(), _capi.as_decision()
    heads = []
    for h in range(8):
        q = torch.from_numpy(asb.fill_uniform(m.n_rows * f, 1 + 3 * h, (m.n_rows, f))).to(dev)
        k = torch.from_numpy(asb.fill_uniform(m.n_cols * f, 2 + 3 * h, (m.n_cols, f))).to(dev)
        v = torch.from_numpy(asb.fill_uniform(m.n_cols * f, 3 + 3 * h, (m.n_cols, f))).to(dev)
        row = {}
        for fused in (1, 0):
            def run():
                asb._check(lib.as_csr_attention_forward(
                    C.byref(cctx), C.byref(ccfg), g.handle, P(q), m.n_rows, P(k), m.n_cols, P(v),
                    m.n_cols, f, f, P(out_t), fused, C.byref(sd), C.byref(pd)))
            t0 = time.perf_counter()
            run()
            torch.cuda.synchronize()
            cold = (time.perf_counter() - t0) * 1e3
            row["fused" if fused else "unfused"] = {"ms": ev_time(run, 3, 1), "first_call_ms": cold}
        heads.append(row)
        del q, k, v
    fused_ms = sum(h["fused"]["ms"] for h in heads)
    unfused_ms = sum(h["unfused"]["ms"] for h in heads)
    by = 4 * m.nnz + 8 * (m.n_rows + 1) + 4 * m.n_rows * f + 4 * m.nnz * f + 4 * m.nnz * f + 4 * m.n_rows * f
    res["c5"] = {"graph": {"n": m.n_rows, "nnz": m.nnz, "F": f, "heads": 8},
                 "sddmm_choice": asb.ScheduleDecision.from_c(sd).choice_string(),
                 "spmm_choice": asb.ScheduleDecision.from_c(pd).choice_string(),
                 "fused_ms_8_heads": fused_ms, "unfused_ms_8_heads": unfused_ms,
                 "fused_gbs": 8 * by / (fused_ms * 1e-3) / 1e9, "heads": heads}
    del keep
    g.close()


def case_bwd(res):
    """Backward pass on the Reddit-shape graph at F=64."""
    import paper_2511_17594_b200.torch_ops  # noqa: F401
    m, _ = bench.make_graph("reddit", 1)
    f = 64
    dev = torch.device("cuda")
    g = asb.Graph.from_csr(m)
    t0 = time.perf_counter()
    gt = g.transpose()
    torch.cuda.synchronize()
    t_transpose = (time.perf_counter() - t0) * 1e3
    t1 = time.perf_counter()
    gt2 = g.transpose()
    torch.cuda.synchronize()
    t_transpose_warm = (time.perf_counter() - t1) * 1e3
    gt2.close()
    dc = torch.from_numpy(asb.fill_uniform(m.n_rows * f, 7, (m.n_rows, f))).to(dev)
    b = torch.from_numpy(asb.fill_uniform(m.n_cols * f, 8, (m.n_cols, f))).to(dev)
    db = torch.empty((m.n_cols, f), dtype=torch.float32, device=dev)
    vals = torch.from_numpy(m.val).to(dev)
    vt = torch.empty_like(vals)
    stream = C.c_void_p(asb.torch_stream_handle())
    hub = asb.variant_from_string("spmm:hubsplit:ft=64:rpc=1:vec=1:hubt=256").to_c()
    asb._check(lib.as_permute_values(gt.handle, P(vals), P(vt), stream))
    t_perm = ev_time(lambda: asb._check(lib.as_permute_values(gt.handle, P(vals), P(vt), stream)))
    t_db = ev_time(lambda: asb._check(lib.as_spmm_values(C.byref(hub), gt.handle, P(vt), P(dc), m.n_rows, f,
                                                         P(db), stream, None)))
    # softmax gradient on probabilities of the graph's own values
    p = torch.empty_like(vals)
    asb._check(lib.as_row_softmax(g.handle, P(vals), P(p), stream))
    gr = torch.from_numpy(asb.fill_uniform(m.nnz, 9, (m.nnz,))).to(dev)
    ds = torch.empty_like(vals)
    t_sm = ev_time(lambda: asb._check(lib.as_row_softmax_backward(g.handle, P(p), P(gr), P(ds), stream)))
    # whole autograd steps through torch.ops (graph + transpose handles cached after the first call)
    crow = torch.from_numpy(m.rowptr.astype(np.int64)).to(dev)
    col = torch.from_numpy(m.colind.astype(np.int32)).to(dev)
    vg, bg = vals.clone().requires_grad_(True), b.clone().requires_grad_(True)
    hv = "spmm:hubsplit:ft=64:rpc=1:vec=1:hubt=256"

    def spmm_step():
        vg.grad = bg.grad = None
        torch.ops.autosage.spmm_csr(crow, col, vg, bg, hv).backward(dc)
    t_spmm_step = ev_time(spmm_step, 3, 1)
    q, k, v = (torch.from_numpy(asb.fill_uniform(m.n_rows * f, 20 + i, (m.n_rows, f))).to(dev).requires_grad_(True)
               for i in range(3))

    def att_step():
        q.grad = k.grad = v.grad = None
        torch.ops.autosage.csr_attention(crow, col, q, k, v, True).backward(dc)
    t_att_step = ev_time(att_step, 3, 1)
    from paper_2511_17594_b200.torch_ops import csr_attention_train

    def att_train_step():
        q.grad = k.grad = v.grad = None
        csr_attention_train(crow, col, q, k, v).backward(dc)
    t_att_train = ev_time(att_train_step, 3, 1)
    n, nnz = m.n_rows, m.nnz
    res["bwd"] = {"graph": {"n": n, "nnz": nnz, "F": f},
                  "transpose_first_ms": t_transpose, "transpose_ms": t_transpose_warm,
                  "permute_ms": t_perm, "permute_gbs": 12 * nnz / (t_perm * 1e-3) / 1e9,
                  "spmm_t_ms": t_db, "spmm_t_gbs": gbs("spmm", n, nnz, f, t_db),
                  "softmax_bwd_ms": t_sm, "softmax_bwd_gbs": (8 * (n + 1) + 12 * nnz) / (t_sm * 1e-3) / 1e9,
                  "spmm_autograd_step_ms": t_spmm_step, "attention_autograd_step_ms": t_att_step,
                  "attention_train_step_ms": t_att_train}
    gt.close()
    g.close()


def case_bf16(res):
    """bf16 dense operand: the same variant on f32 and bf16 B."""
    out = {}
    for cfg, fs, variant in (("reddit", (32, 64, 128), "spmm:hubsplit:ft=64:rpc=1:vec=1:hubt=256"),
                             ("products", (100,), "spmm:hubsplit:ft=64:rpc=1:vec=1:hubt=256")):
        m, _ = bench.make_graph(cfg, 1)
        g = asb.Graph.from_csr(m)
        dev = torch.device("cuda")
        stream = C.c_void_p(asb.torch_stream_handle())
        cv = asb.variant_from_string(variant).to_c()
        for f in fs:
            b = torch.from_numpy(asb.fill_uniform(m.n_cols * f, 1 + f, (m.n_cols, f))).to(dev)
            b16 = b.to(torch.bfloat16)
            c = torch.empty((m.n_rows, f), dtype=torch.float32, device=dev)
            t32 = ev_time(lambda: asb._check(lib.as_spmm(C.byref(cv), g.handle, P(b), m.n_cols, f, P(c), stream,
                                                         None)))
            t16 = ev_time(lambda: asb._check(lib.as_spmm_bf16(C.byref(cv), g.handle, None, P(b16), m.n_cols, f,
                                                              P(c), stream, None)))
            # bf16 gather-model bytes: the B gather term at 2 bytes per element
            by16 = 8 * m.nnz + 2 * m.nnz * f + 4 * m.n_rows * f + 8 * (m.n_rows + 1)
            out[f"{cfg}_F{f}"] = {"variant": variant, "f32_ms": t32, "bf16_ms": t16, "speedup": t32 / t16,
                                  "f32_gbs": gbs("spmm", m.n_rows, m.nnz, f, t32),
                                  "bf16_gbs": by16 / (t16 * 1e-3) / 1e9}
            if cfg == "reddit" and f in (32, 64):
                x = torch.from_numpy(asb.fill_uniform(m.n_rows * f, 2 + f, (m.n_rows, f))).to(dev)
                y = torch.from_numpy(asb.fill_uniform(m.n_cols * f, 3 + f, (m.n_cols, f))).to(dev)
                x16, y16 = x.to(torch.bfloat16), y.to(torch.bfloat16)
                sv = torch.empty(m.nnz, dtype=torch.float32, device=dev)
                sd = asb.variant_from_string("sddmm:rowparallel:ft=32:rpc=1:vec=0:hubt=256").to_c()
                s32 = ev_time(lambda: asb._check(lib.as_sddmm(C.byref(sd), g.handle, P(x), m.n_rows, P(y), m.n_cols,
                                                              f, P(sv), stream, None)))
                s16 = ev_time(lambda: asb._check(lib.as_sddmm_bf16(C.byref(sd), g.handle, P(x16), m.n_rows, P(y16),
                                                                   m.n_cols, f, P(sv), stream, None)))
                out[f"{cfg}_F{f}_sddmm"] = {"variant": "sddmm:rowparallel:ft=32:rpc=1:vec=0:hubt=256",
                                            "f32_ms": s32, "bf16_ms": s16, "speedup": s32 / s16,
                                            "f32_gbs": gbs("sddmm", m.n_rows, m.nnz, f, s32),
                                            "bf16_gbs": (8 * m.nnz + 4 * m.nnz * f + 4 * m.nnz) / (s16 * 1e-3) / 1e9}
                if f == 64:
                    # one attention head through the torch op: f32 staged vs bf16 q, k, v
                    import paper_2511_17594_b200.torch_ops  # noqa: F401
                    crow = torch.from_numpy(m.rowptr.astype(np.int64)).to(dev)
                    col = torch.from_numpy(m.colind.astype(np.int32)).to(dev)
                    att = torch.ops.autosage.csr_attention
                    a32 = ev_time(lambda: att(crow, col, x, y, b, False))
                    a16 = ev_time(lambda: att(crow, col, x16, y16, b16, False))
                    out[f"{cfg}_F{f}_attention"] = {"f32_staged_ms": a32, "bf16_ms": a16, "speedup": a32 / a16}
                    del crow, col
                del x, y, x16, y16, sv
            del b, b16, c
        g.close()
    res["bf16"] = out


def run_meta():
    """Reproducibility sidecar (the reference bench's .meta.json fields,
    proj/tools/autosage_bench.cpp:144-165, re-targeted): device signature as
    folded into schedule-cache keys, host CPU and cores for the CPU reference,
    toolchain, driver and library versions."""
    import platform
    import subprocess
    dp = asb.DeviceProfile.gpu()
    cpu = ""
    try:
        with open("/proc/cpuinfo") as fh:
            cpu = next((ln.split(":", 1)[1].strip() for ln in fh if ln.startswith("model name")), "")
    except OSError:
        pass
    try:
        drv = subprocess.run(["nvidia-smi", "--query-gpu=driver_version,clocks.max.sm", "--format=csv,noheader"],
                             capture_output=True, text=True, timeout=20).stdout.strip()
    except Exception:
        drv = ""
    return {"device_sig": dp.device_sig, "bw_eff_gbs": dp.bw_eff / 1e9, "flops_eff_gflops": dp.flops_eff / 1e9,
            "sms": dp.cores, "cost_model": "b200" if dp.model == 1 else "reference",
            "host_cpu": cpu, "host_cores": os.cpu_count(), "python": platform.python_version(),
            "torch": torch.__version__, "cuda_runtime": torch.version.cuda, "driver_and_max_sm_clock": drv,
            "probe_config": dataclasses_asdict(asb.ProbeConfig.from_env()),
            "toolchain": asb.toolchain_tag() if hasattr(asb, "toolchain_tag") else None}


def dataclasses_asdict(x):
    import dataclasses
    return dataclasses.asdict(x)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cases", default="c1,c2,c3,c4,c5")
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "sweep.json"))
    a = ap.parse_args()
    res = {"gpu": torch.cuda.get_device_name(), "peak_gbs": PEAK, "meta": run_meta()}
    for cs in a.cases.split(","):
        t0 = time.time()
        globals()[f"case_{cs}"](res)
        print(cs, "done in", round(time.time() - t0, 1), "s", flush=True)
        with open(a.out, "w") as fh:
            json.dump(res, fh, indent=1)


if __name__ == "__main__":
    main()
