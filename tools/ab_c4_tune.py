#!/usr/bin/env python3
"""c4 skew graphs at F=64 (B = 282 MB, gathered from HBM): SpMM time of the
hub-split variant under one AUTOSAGE_DEV_SPMM_TUNE setting (entries in flight
per lane group x register cap), L2 flushed before each call.  One process
per setting (the knob is read once):
  for t in default 8x96 ...; do AUTOSAGE_DEV_SPMM_TUNE=$t python tools/ab_c4_tune.py; done"""
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
    tune = os.environ.get("AUTOSAGE_DEV_SPMM_TUNE", "default")
    s = asb.torch_stream_handle()
    flush = torch.empty(64 << 20, device="cuda")
    out = []
    for alpha in (2.0, 2.5, 3.0):
        m = bench.with_hubs(asb.gen_powerlaw(1_100_000, 1_100_000, 24_000_000, alpha, 4, 1_000_000, 7),
                            [1_000_000, 250_000, 60_000], 11)
        g = asb.Graph.from_csr(m)
        f = 64
        b = torch.from_numpy(asb.fill_uniform(m.n_cols * f, 1 + f, (m.n_cols, f))).cuda()
        c = torch.empty((m.n_rows, f), device="cuda")
        for vs in ("spmm:hubsplit:ft=64:rpc=1:vec=1:hubt=256",):
            v = asb.variant_from_string(vs).to_c()

            def run():
                asb._check(_capi.lib.as_spmm(C.byref(v), g.handle, C.c_void_p(b.data_ptr()), m.n_cols, f,
                                             C.c_void_p(c.data_ptr()), C.c_void_p(s), None))
            run()
            ts = []
            for _ in range(9):
                flush.zero_()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                run()
                e1.record()
                e1.synchronize()
                ts.append(e0.elapsed_time(e1))
            ms = sorted(ts)[4]
            gbs = bench.gather_bytes("spmm", m.n_rows, m.nnz, f) / (ms * 1e-3) / 1e9
            out.append(f"a={alpha} {ms:.3f} ms {gbs:.0f} GB/s")
        g.close()
        del b, c
    print(f"tune={tune}: " + "  ".join(out), flush=True)


if __name__ == "__main__":
    main()
