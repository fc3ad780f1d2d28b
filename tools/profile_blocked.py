#!/usr/bin/env python3
"""Column-blocked SpMM cost on one GPU (the compute side of dist.py
blocked_spmm): rank 0's nnz-balanced shard of a g-way split, padded layout,
unblocked (as_spmm, decided variant) vs blocked in 1 / 2 / g column blocks.
The exchange itself needs g GPUs; with the measured per-block times the
overlap can be modelled against the NVLink all-gather time.
  python tools/profile_blocked.py --config products --world 8"""
import argparse
import ctypes as C
import json
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


def ev_time(fn, reps=10, flush=None):
    ts = []
    for _ in range(reps + 2):
        if flush is not None:
            flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    ts = sorted(ts[2:])
    return ts[len(ts) // 2]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="products")
    ap.add_argument("--world", type=int, default=8)
    ap.add_argument("--rank", type=int, default=0)
    ap.add_argument("--variant", default="spmm:hubsplit:ft=128:rpc=1:vec=1:hubt=256")
    a = ap.parse_args()
    m, f = bench.make_graph(a.config, 1)
    sh = RowSharding(m.rowptr, a.world, a.rank)
    pg = sh.shard_graph_host(m)
    g = asb.Graph.from_csr(pg)
    b = asb.fill_uniform(m.n_cols * f, 1 + f, (m.n_cols, f))
    pad = np.zeros((sh.padded_rows, f), np.float32)
    pad[sh.perm] = b
    bd = torch.from_numpy(pad).cuda()
    c = torch.empty((pg.n_rows, f), device="cuda")
    flush = torch.empty(64 << 20, device="cuda")
    v = asb.variant_from_string(a.variant)
    cv = v.to_c()
    s = asb.torch_stream_handle()
    res = {"config": a.config, "world": a.world, "rank": a.rank, "rows": pg.n_rows, "nnz": pg.nnz, "F": f,
           "variant": a.variant}

    def plain():
        asb._check(_capi.lib.as_spmm(C.byref(cv), g.handle, C.c_void_p(bd.data_ptr()), bd.shape[0], f,
                                     C.c_void_p(c.data_ptr()), C.c_void_p(s), None))
    res["unblocked_ms"] = ev_time(plain, flush=flush)
    want = None
    plain()
    torch.cuda.synchronize()
    want = c.cpu().numpy().copy()
    for groups in sorted({1, 2, a.world}):
        p = asb.BlockedSpmm(g, v, sh.column_cuts(groups))

        def blocked():
            for k in range(p.n_blocks):
                p.run(k, bd, c)
        t = ev_time(blocked, flush=flush)
        per = []
        for k in range(p.n_blocks):
            per.append(ev_time(lambda: p.run(k, bd, c) if k else p.run(0, bd, c), reps=5))
        blocked()
        torch.cuda.synchronize()
        same = bool(np.array_equal(c.cpu().numpy().view(np.uint32), want.view(np.uint32)))
        res[f"blocked_{groups}"] = {"ms": t, "per_block_ms": per, "bit_identical": same}
        p.close()
    # NVLink model: each rank receives (world-1)/world of B at the measured
    # 770 GB/s peer rate (B200_PROFILING.md)
    recv = (a.world - 1) * sh.shard * f * 4
    res["gather_model_ms"] = recv / 770e9 * 1e3
    print(json.dumps(res))


if __name__ == "__main__":
    main()
