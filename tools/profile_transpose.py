"""Time the device transpose (backward setup) on the Reddit-shape graph:
wall clock per call, and (under ncu) its kernel launches.

  python tools/profile_transpose.py [--reps 3]
"""
import argparse
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
import paper_2511_17594_b200 as asb  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--config", default="reddit")
    a = ap.parse_args()
    m, _ = bench.make_graph(a.config, 1)
    g = asb.Graph.from_csr(m)
    for i in range(a.reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        gt = g.transpose()
        torch.cuda.synchronize()
        print(f"transpose {i}: {(time.perf_counter() - t0) * 1e3:.1f} ms", flush=True)
        gt.close()


if __name__ == "__main__":
    main()
