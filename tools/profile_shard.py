#!/usr/bin/env python3
"""Time SpMM variants on one nnz-balanced row shard of a bench config (the
per-rank compute of a g-GPU step), for ncu capture.
  python tools/profile_shard.py --config products --world 8 --rank 0"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2511_17594_b200 as asb  # noqa: E402
from paper_2511_17594_b200.dist import RowSharding  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="products")
    ap.add_argument("--world", type=int, default=8)
    ap.add_argument("--rank", type=int, default=0)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--spmm", default="spmm:hubsplit:ft=128:rpc=4:vec=1:hubt=256")
    a = ap.parse_args()
    m, f = bench.make_graph(a.config, 1)
    sh = RowSharding(m.rowptr, a.world, a.rank)
    full = asb.Graph.from_csr(m)
    g = full.row_range(sh.r0, sh.r1) if a.world > 1 else full
    b = torch.from_numpy(asb.fill_uniform(m.n_cols * f, 1 + f, (m.n_cols, f))).cuda()
    for spec in a.spmm.split(","):
        v = asb.variant_from_string(spec)
        for _ in range(a.reps):
            r = asb.dispatch(v, g, b)
            torch.cuda.synchronize()
            print(a.config, f"g={a.world}", f"rank={a.rank}", spec, r.elapsed_ms, flush=True)


if __name__ == "__main__":
    main()
