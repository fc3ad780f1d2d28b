#!/usr/bin/env python3
"""f32 vs bf16 vs f16 operands on Reddit-shape (F=64): SpMM (hub-split),
SDDMM (scalar order) and one head of CSR attention, fused and staged, through
the torch ops (CUDA events, L2 flushed before each call, median of 7)."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2511_17594_b200 as asb  # noqa: E402
import paper_2511_17594_b200.torch_ops  # noqa: E402,F401

SPMM = "spmm:hubsplit:ft=64:rpc=1:vec=1:hubt=256"
SDDMM = "sddmm:rowparallel:ft=32:rpc=1:vec=0:hubt=256"


def ev(fn, flush, reps=7):
    fn()
    ts = []
    for _ in range(reps):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    return sorted(ts)[len(ts) // 2]


def main():
    m, f = bench.make_graph("reddit", 1)
    dev = torch.device("cuda")
    crow = torch.from_numpy(m.rowptr.astype(np.int64)).to(dev)
    col = torch.from_numpy(m.colind.astype(np.int32)).to(dev)
    val = torch.from_numpy(m.val).to(dev)
    empty = torch.empty(0, device=dev)
    b, x, y = (torch.from_numpy(a).to(dev) for a in bench.dense_inputs(asb.fill_uniform, m, f, 1))
    flush = torch.empty(64 << 20, device=dev)
    ops = torch.ops.autosage
    res = {}
    for name, dt in (("f32", torch.float32), ("bf16", torch.bfloat16), ("f16", torch.float16)):
        bb, xx, yy = b.to(dt), x.to(dt), y.to(dt)
        r = {"spmm_ms": ev(lambda: ops.spmm_csr(crow, col, val, bb, SPMM), flush),
             "sddmm_ms": ev(lambda: ops.sddmm_csr(crow, col, xx, yy, SDDMM), flush)}
        if dt == torch.float32:
            r["attention_fused_ms"] = ev(lambda: ops.csr_attention(crow, col, xx, yy, bb, True), flush)
            r["attention_staged_ms"] = ev(lambda: ops.csr_attention(crow, col, xx, yy, bb, False), flush)
        else:
            r["attention_fused_ms"] = ev(lambda: ops.csr_attention(crow, col, xx, yy, bb, True), flush)
            r["attention_staged_ms"] = ev(lambda: ops.csr_attention(crow, col, xx, yy, bb, False), flush)
        res[name] = r
        print(name, json.dumps(r), flush=True)
    print(json.dumps(res))


if __name__ == "__main__":
    main()
