#!/usr/bin/env python3
"""Time the CSR row softmax (as_row_softmax, device values) on a bench config."""
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
    ap.add_argument("--reps", type=int, default=5)
    a = ap.parse_args()
    m, _ = bench.make_graph(a.config, 1)
    g = asb.Graph.from_csr(m)
    dev = torch.device("cuda")
    vin = torch.from_numpy(asb.fill_uniform(m.nnz, 9, (m.nnz,))).to(dev)
    vout = torch.empty_like(vin)
    stream = C.c_void_p(asb.torch_stream_handle())
    for _ in range(a.reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        asb._check(_capi.lib.as_row_softmax(g.handle, C.c_void_p(vin.data_ptr()), C.c_void_p(vout.data_ptr()),
                                            stream))
        e1.record()
        e1.synchronize()
        print("row_softmax", a.config, e0.elapsed_time(e1), flush=True)


if __name__ == "__main__":
    main()
