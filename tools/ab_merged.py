#!/usr/bin/env python3
"""Hub-split SpMM as one launch over pieces + light rows
(AUTOSAGE_DEV_SPMM_MERGED=1) vs light rows and pieces as two kernels on
forked streams (default).  One process per setting (the knob is read once);
prints times and a bit checksum of every output, which must match across
the two settings.
  for m in 0 1; do AUTOSAGE_DEV_SPMM_MERGED=$m python tools/ab_merged.py; done"""
import ctypes as C
import hashlib
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2511_17594_b200 as asb  # noqa: E402
from paper_2511_17594_b200 import _capi  # noqa: E402
from paper_2511_17594_b200.dist import RowSharding  # noqa: E402


def timed(g, m_cols, f, vs, b, c, s, flush, reps=9):
    v = asb.variant_from_string(vs).to_c()

    def run():
        asb._check(_capi.lib.as_spmm(C.byref(v), g.handle, C.c_void_p(b.data_ptr()), m_cols, f,
                                     C.c_void_p(c.data_ptr()), C.c_void_p(s), None))
    run()
    evs = []
    for _ in range(reps):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        run()
        e1.record()
        evs.append((e0, e1))
    torch.cuda.synchronize()
    ts = sorted(e0.elapsed_time(e1) for e0, e1 in evs)
    h = hashlib.sha1(c.view(torch.int32).cpu().numpy().tobytes()).hexdigest()[:10]
    return ts[len(ts) // 2], h


def main():
    tag = os.environ.get("AUTOSAGE_DEV_SPMM_MERGED", "0")
    s = asb.torch_stream_handle()
    flush = torch.empty(64 << 20, device="cuda")
    out = []
    cases = [("reddit", 64, "spmm:hubsplit:ft=64:rpc=1:vec=1:hubt=256", 1),
             ("reddit", 128, "spmm:hubsplit:ft=128:rpc=1:vec=1:hubt=256", 1),
             ("products", 100, "spmm:hubsplit:ft=128:rpc=1:vec=1:hubt=256", 1),
             ("products", 100, "spmm:hubsplit:ft=128:rpc=1:vec=1:hubt=256", 8)]
    graphs = {}
    for cfg, f, vs, world in cases:
        if cfg not in graphs:
            graphs.clear()
            graphs[cfg] = bench.make_graph(cfg, 1)[0]
        m = graphs[cfg]
        if world > 1:
            sh = RowSharding(m.rowptr, world, 0)
            gm = sh.shard_graph_host(m)
        else:
            gm = m
        g = asb.Graph.from_csr(gm)
        b = torch.from_numpy(asb.fill_uniform(gm.n_cols * f, 1 + f, (gm.n_cols, f))).cuda()
        c = torch.empty((gm.n_rows, f), device="cuda")
        ms, h = timed(g, gm.n_cols, f, vs, b, c, s, flush)
        out.append(f"{cfg}/{world} F={f} {ms:.3f} ms [{h}]")
        g.close()
        del b, c
    for alpha in (2.0, 3.0):
        m = bench.with_hubs(asb.gen_powerlaw(1_100_000, 1_100_000, 24_000_000, alpha, 4, 1_000_000, 7),
                            [1_000_000, 250_000, 60_000], 11)
        g = asb.Graph.from_csr(m)
        f = 64
        b = torch.from_numpy(asb.fill_uniform(m.n_cols * f, 1 + f, (m.n_cols, f))).cuda()
        c = torch.empty((m.n_rows, f), device="cuda")
        ms, h = timed(g, m.n_cols, f, "spmm:hubsplit:ft=64:rpc=1:vec=1:hubt=256", b, c, s, flush)
        out.append(f"c4 a={alpha} F=64 {ms:.3f} ms [{h}]")
        g.close()
    print(f"merged={tag}: " + "  ".join(out), flush=True)


if __name__ == "__main__":
    main()
