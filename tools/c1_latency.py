#!/usr/bin/env python3
"""c1 latency breakdown: GPU event time per op (back-to-back, L2 flushed or
not), host enqueue time per call, and the same op via as_spmm (fixed variant)
vs as_spmm_auto (decide cache hit each call).
  python tools/c1_latency.py [--config c1] [--reps 200]"""
import argparse
import ctypes as C
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2511_17594_b200 as asb  # noqa: E402
from paper_2511_17594_b200 import _capi  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c1")
    ap.add_argument("--reps", type=int, default=200)
    a = ap.parse_args()
    m, f = bench.make_graph(a.config, 1)
    b, x, y = bench.dense_inputs(asb.fill_uniform, m, f, 1)
    g = asb.Graph.from_csr(m)
    dev = torch.device("cuda")
    bd, xd, yd = (torch.from_numpy(t).to(dev) for t in (b, x, y))
    c = torch.empty((m.n_rows, f), device=dev)
    sv = torch.empty(m.nnz, device=dev)
    flush = torch.empty(64 << 20, dtype=torch.float32, device=dev)
    lib = _capi.lib
    stream = asb.torch_stream_handle(dev)
    cache = asb.ScheduleCache()
    ctx = asb.ScheduleContext(cache=cache, stream=stream)
    cctx, keep = ctx.to_c()
    ccfg = asb.ProbeConfig.from_env().to_c()
    d = _capi.as_decision()
    P = lambda t: C.c_void_p(t.data_ptr())  # noqa: E731

    def spmm_auto():
        asb._check(lib.as_spmm_auto(C.byref(cctx), C.byref(ccfg), g.handle, P(bd), m.n_cols, f, P(c), C.byref(d)))

    def sddmm_auto():
        asb._check(lib.as_sddmm_auto(C.byref(cctx), C.byref(ccfg), g.handle, P(xd), m.n_rows, P(yd), m.n_cols, f,
                                     P(sv), C.byref(d)))
    spmm_auto()
    sddmm_auto()
    torch.cuda.synchronize()
    choice_s = asb.ScheduleDecision.from_c(d)
    spmm_auto()
    choice_p = asb.ScheduleDecision.from_c(d)
    vs = choice_p.choice.to_c() if choice_p.choice else None
    vd = None

    def spmm_fixed():
        asb._check(lib.as_spmm(C.byref(vs) if vs else None, g.handle, P(bd), m.n_cols, f, P(c), C.c_void_p(stream),
                               None))

    res = {}
    for name, fn in (("spmm_auto", spmm_auto), ("spmm_fixed", spmm_fixed), ("sddmm_auto", sddmm_auto)):
        for cold in (False, True):
            evs = []
            host = []
            for _ in range(a.reps):
                if cold:
                    flush.zero_()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                t0 = time.perf_counter()
                fn()
                host.append(time.perf_counter() - t0)
                e1.record()
                evs.append((e0, e1))
            torch.cuda.synchronize()
            ts = sorted(e0.elapsed_time(e1) for e0, e1 in evs)
            hs = sorted(host)
            res[f"{name}{'_cold' if cold else '_warm'}"] = (ts[len(ts) // 2], hs[len(hs) // 2] * 1e3)
        # back-to-back throughput: many calls, one pair of events
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(a.reps):
            fn()
        e1.record()
        torch.cuda.synchronize()
        res[f"{name}_b2b"] = (e0.elapsed_time(e1) / a.reps, None)
    print("choices", choice_p.choice_string(), choice_s.choice_string())
    for k, (gpu_ms, host_ms) in res.items():
        print(f"{k:18s} gpu(event) {gpu_ms:.4f} ms   host enqueue {host_ms if host_ms is None else round(host_ms, 4)} ms")
    del keep


if __name__ == "__main__":
    main()
