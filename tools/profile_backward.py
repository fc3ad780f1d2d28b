"""One forward + backward step of torch.ops.autosage.spmm_csr and of
csr_attention (fused) on the Reddit-shape graph at F=64, for an ncu launch
list (the handles and the transpose are built in an untimed first step):

  python tools/profile_backward.py --store gpurun_out/bwd.cache     # decide without ncu
  ncu --metrics gpu__time_duration.sum --clock-control none --csv \\
      --log-file gpurun_out/bwd_launches.csv python tools/profile_backward.py --load gpurun_out/bwd.cache

(Probe timings taken under ncu are serialised and distorted, so the decisions
are made in a plain run and replayed from the stored cache under ncu.)
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2511_17594_b200 as asb  # noqa: E402
import paper_2511_17594_b200.torch_ops  # noqa: E402,F401


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--store", default="")
    ap.add_argument("--load", default="")
    a = ap.parse_args()
    import paper_2511_17594_b200.torch_ops as T
    T._CACHE = asb.ScheduleCache()
    if a.load:
        T._CACHE.load(a.load)
    m, _ = bench.make_graph("reddit", 1)
    f = 64
    dev = torch.device("cuda")
    crow = torch.from_numpy(m.rowptr.astype(np.int64)).to(dev)
    col = torch.from_numpy(m.colind.astype(np.int32)).to(dev)
    val = torch.from_numpy(m.val).to(dev).requires_grad_(True)
    b = torch.from_numpy(asb.fill_uniform(m.n_cols * f, 8, (m.n_cols, f))).to(dev).requires_grad_(True)
    dc = torch.from_numpy(asb.fill_uniform(m.n_rows * f, 7, (m.n_rows, f))).to(dev)
    q, k, v = (torch.from_numpy(asb.fill_uniform(m.n_rows * f, 20 + i, (m.n_rows, f))).to(dev).requires_grad_(True)
               for i in range(3))
    hv = "spmm:hubsplit:ft=64:rpc=1:vec=1:hubt=256"
    for step in range(2):  # step 0 builds handles, transpose, decisions
        torch.cuda.nvtx.range_push(f"spmm_step{step}")
        torch.ops.autosage.spmm_csr(crow, col, val, b, hv).backward(dc)
        torch.cuda.synchronize()
        torch.cuda.nvtx.range_pop()
        torch.cuda.nvtx.range_push(f"attention_step{step}")
        torch.ops.autosage.csr_attention(crow, col, q, k, v, True).backward(dc)
        torch.cuda.synchronize()
        torch.cuda.nvtx.range_pop()
    if a.store:
        T._CACHE.store(a.store)
    print("ok")


if __name__ == "__main__":
    main()
