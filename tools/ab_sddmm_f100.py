#!/usr/bin/env python3
"""F=100 pair-kernel A/B on the Products-shape graph:
general chunk kernel (AUTOSAGE_DEV_SDDMM_PAIR=0) vs the 25-unit-pitch pair
kernel (=1), fixed variants, L2 flushed before each call; the two
outputs must be bit-identical on the full graph.
  python tools/ab_sddmm_f100.py [--config products] [--reps 7]"""
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
    ap.add_argument("--config", default="products")
    ap.add_argument("--reps", type=int, default=7)
    ap.add_argument("--fs", default="100")
    a = ap.parse_args()
    m, _ = bench.make_graph(a.config, 1)
    g = asb.Graph.from_csr(m.with_values(None))
    s = asb.torch_stream_handle()
    flush = torch.empty(64 << 20, device="cuda")
    out = torch.empty(m.nnz, device="cuda")
    for f in (int(v) for v in a.fs.split(",")):
        x = torch.from_numpy(asb.fill_uniform(m.n_rows * f, 1 + f, (m.n_rows, f))).cuda()
        y = torch.from_numpy(asb.fill_uniform(m.n_cols * f, 2 + f, (m.n_cols, f))).cuda()
        for vs in ("sddmm:rowparallel:ft=32:rpc=1:vec=0:hubt=256", "sddmm:rowparallel:ft=32:rpc=1:vec=1:hubt=256",
                   "sddmm:rowparallel:ft=64:rpc=1:vec=1:hubt=256"):
            v = asb.variant_from_string(vs).to_c()

            def run():
                asb._check(_capi.lib.as_sddmm(C.byref(v), g.handle, C.c_void_p(x.data_ptr()), m.n_rows,
                                              C.c_void_p(y.data_ptr()), m.n_cols, f, C.c_void_p(out.data_ptr()),
                                              C.c_void_p(s), None))
            res, outs = {}, {}
            for pm in ("0", "1", "0", "1"):
                os.environ["AUTOSAGE_DEV_SDDMM_PAIR"] = pm
                run()
                ts = []
                for _ in range(a.reps):
                    flush.zero_()
                    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    e0.record()
                    run()
                    e1.record()
                    e1.synchronize()
                    ts.append(e0.elapsed_time(e1))
                res.setdefault(pm, []).append(sorted(ts)[len(ts) // 2])
                outs[pm] = out.clone()
            same = torch.equal(outs["0"].view(torch.int32), outs["1"].view(torch.int32))
            print(f"F={f} {vs.split(':', 2)[2][:14]:14s} chunk {min(res['0']):.3f} ms  pair "
                  f"{min(res['1']):.3f} ms  bit-identical={same}", flush=True)
            del outs
        del x, y


if __name__ == "__main__":
    main()
