#!/usr/bin/env python3
"""Run chosen SpMM / SDDMM variants on a bench config's full graph, a few
times each, for ncu capture (no probes, so `-k regex:... -s 1 -c 1` lands on
a steady-state full-graph launch).

  python tools/profile_kernels.py --config reddit \
      --spmm spmm:hubsplit:ft=32:rpc=4:vec=1:hubt=256 \
      --sddmm sddmm:hubsplit:ft=32:rpc=4:vec=1:hubt=256 --reps 3
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
import paper_2511_17594_b200 as asb  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="reddit")
    ap.add_argument("--f", type=int, default=0)
    ap.add_argument("--spmm", default="")
    ap.add_argument("--sddmm", default="")
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--seed", type=int, default=1)
    a = ap.parse_args()
    m, f = bench.make_graph(a.config, a.seed)
    f = a.f or f
    g = asb.Graph.from_csr(m)
    b = torch.from_numpy(asb.fill_uniform(m.n_cols * f, a.seed + f, (m.n_cols, f))).cuda()
    x = torch.from_numpy(asb.fill_uniform(m.n_rows * f, a.seed + f, (m.n_rows, f))).cuda()
    y = torch.from_numpy(asb.fill_uniform(m.n_cols * f, a.seed + f + 1, (m.n_cols, f))).cuda()
    for spec in filter(None, a.spmm.split(",")):
        v = asb.variant_from_string(spec) if spec != "baseline" else None
        for _ in range(a.reps):
            r = asb.dispatch(v, g, b) if v else None
            if v is None:
                asb.spmm_baseline(g, b)
            torch.cuda.synchronize()
            print(spec, r.elapsed_ms if r else "", flush=True)
    for spec in filter(None, a.sddmm.split(",")):
        v = asb.variant_from_string(spec) if spec != "baseline" else None
        for _ in range(a.reps):
            r = asb.dispatch(v, g, x, y) if v else None
            if v is None:
                asb.sddmm_baseline(g, x, y)
            torch.cuda.synchronize()
            print(spec, r.elapsed_ms if r else "", flush=True)


if __name__ == "__main__":
    main()
