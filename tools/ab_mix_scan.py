#!/usr/bin/env python3
"""Finite-scan cap A/B (AUTOSAGE_DEV_MIX_SCAN_MB): dense operands above the
cap skip the Inf/NaN scan and widen every component with F2F on the XU
pipe; below it, a finite operand lets the kernels re-bias half the
components on the ALU instead.  Same variant, same output bits.
  python tools/ab_mix_scan.py [--reps 7]"""
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

CASES = {
    "reddit": [(128, "spmm:hubsplit:ft=128:rpc=1:vec=1:hubt=256", "sddmm:rowparallel:ft=32:rpc=1:vec=0:hubt=256"),
               (256, "spmm:hubsplit:ft=128:rpc=1:vec=1:hubt=256", "sddmm:rowparallel:ft=32:rpc=1:vec=0:hubt=256")],
    "products": [(100, "spmm:hubsplit:ft=128:rpc=1:vec=1:hubt=256", "sddmm:rowparallel:ft=64:rpc=1:vec=1:hubt=256")],
}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=7)
    ap.add_argument("--configs", default="reddit,products")
    a = ap.parse_args()
    s = asb.torch_stream_handle()
    flush = torch.empty(64 << 20, device="cuda")
    lib = _capi.lib
    for cfg in a.configs.split(","):
        m, _ = bench.make_graph(cfg, 1)
        g = asb.Graph.from_csr(m)
        out = torch.empty(m.nnz, device="cuda")
        for f, vsp, vsd in CASES[cfg]:
            b = torch.from_numpy(asb.fill_uniform(m.n_cols * f, 1 + f, (m.n_cols, f))).cuda()
            x = torch.from_numpy(asb.fill_uniform(m.n_rows * f, 1 + f, (m.n_rows, f))).cuda()
            y = torch.from_numpy(asb.fill_uniform(m.n_cols * f, 2 + f, (m.n_cols, f))).cuda()
            c = torch.empty((m.n_rows, f), device="cuda")
            for op, vs in (("spmm", vsp), ("sddmm", vsd)):
                v = asb.variant_from_string(vs).to_c()
                if op == "spmm":
                    def run():
                        asb._check(lib.as_spmm(C.byref(v), g.handle, C.c_void_p(b.data_ptr()), m.n_cols, f,
                                               C.c_void_p(c.data_ptr()), C.c_void_p(s), None))
                    res_t = c
                else:
                    def run():
                        asb._check(lib.as_sddmm(C.byref(v), g.handle, C.c_void_p(x.data_ptr()), m.n_rows,
                                                C.c_void_p(y.data_ptr()), m.n_cols, f, C.c_void_p(out.data_ptr()),
                                                C.c_void_p(s), None))
                    res_t = out
                res, ref = {}, None
                for cap in ("96", "4096") * 2:
                    os.environ["AUTOSAGE_DEV_MIX_SCAN_MB"] = cap
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
                    res.setdefault(cap, []).append(sorted(ts)[len(ts) // 2])
                    if ref is None:
                        ref = res_t.clone()
                    same = torch.equal(ref.view(torch.int32), res_t.view(torch.int32))
                    assert same, (cfg, f, op, cap)
                print(f"{cfg} F={f} {op:5s} {vs.split(':', 1)[1][:24]:24s} no-scan {min(res['96']):.3f} ms  "
                      f"scan+mix {min(res['4096']):.3f} ms  bit-identical=True", flush=True)
            del b, x, y, c
        g.close()
        del out


if __name__ == "__main__":
    main()
