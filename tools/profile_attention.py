#!/usr/bin/env python3
"""Run CSR attention (fused or unfused) on a bench config graph for ncu capture.
  python tools/profile_attention.py --config reddit --fused 1 --reps 3"""
import argparse
import ctypes as C
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2511_17594_b200 as asb  # noqa: E402
from paper_2511_17594_b200 import _capi  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="reddit")
    ap.add_argument("--f", type=int, default=64)
    ap.add_argument("--fused", type=int, default=1)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--cache", default="", help="schedule cache: load if present, store after the run")
    ap.add_argument("--replay-only", action="store_true", help="decisions must come from --cache")
    a = ap.parse_args()
    m, _ = bench.make_graph(a.config, 1)
    f = a.f
    g = asb.Graph.from_csr(m)
    dev = torch.device("cuda")
    q = torch.from_numpy(asb.fill_uniform(m.n_rows * f, 1, (m.n_rows, f))).to(dev)
    k = torch.from_numpy(asb.fill_uniform(m.n_cols * f, 2, (m.n_cols, f))).to(dev)
    v = torch.from_numpy(asb.fill_uniform(m.n_cols * f, 3, (m.n_cols, f))).to(dev)
    out = torch.empty((m.n_rows, f), dtype=torch.float32, device=dev)
    cache = asb.ScheduleCache()
    if a.cache and os.path.exists(a.cache):
        cache.load(a.cache)
    ctx = asb.ScheduleContext(cache=cache, stream=asb.torch_stream_handle(),
                              replay=asb.ReplayPolicy(replay_only=a.replay_only, strict=a.replay_only))
    cctx, keep = ctx.to_c()
    ccfg = asb.ProbeConfig.from_env().to_c()
    sd, pd = _capi.as_decision(), _capi.as_decision()
    P = lambda t: C.c_void_p(t.data_ptr())  # noqa: E731
    for i in range(a.reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        asb._check(_capi.lib.as_csr_attention_forward(C.byref(cctx), C.byref(ccfg), g.handle, P(q), m.n_rows,
                                                      P(k), m.n_cols, P(v), m.n_cols, f, f, P(out), a.fused,
                                                      C.byref(sd), C.byref(pd)))
        e1.record()
        e1.synchronize()
        print("attention fused=%d" % a.fused, e0.elapsed_time(e1), flush=True)
    print("choices", asb.ScheduleDecision.from_c(sd).choice_string(), asb.ScheduleDecision.from_c(pd).choice_string())
    if a.cache and not a.replay_only:
        cache.store(a.cache)
    del keep


if __name__ == "__main__":
    main()
