#!/usr/bin/env python3
"""L2 policy of the widened-X staging in the SDDMM pair kernels
(AUTOSAGE_DEV_SDDMM_XPOL: 0 = as Y (evict_last when Y fits), 1 = normal,
2 = evict_first), Reddit-shape, the sequential variant the scheduler picks,
F = 64 (single launch) and 128 / 256 (pass-major); L2 flushed before each
call, interleaved repeats; outputs must not change.
  python tools/ab_sddmm_xpol.py [--fs 64,128,256]"""
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
    ap.add_argument("--reps", type=int, default=7)
    ap.add_argument("--fs", default="64,128,256")
    a = ap.parse_args()
    m, _ = bench.make_graph(a.config, 1)
    g = asb.Graph.from_csr(m.with_values(None))
    s = asb.torch_stream_handle()
    flush = torch.empty(64 << 20, device="cuda")
    out = torch.empty(m.nnz, device="cuda")
    v = asb.variant_from_string("sddmm:rowparallel:ft=32:rpc=1:vec=0:hubt=256").to_c()
    for f in (int(t) for t in a.fs.split(",")):
        x = torch.from_numpy(asb.fill_uniform(m.n_rows * f, 1 + f, (m.n_rows, f))).cuda()
        y = torch.from_numpy(asb.fill_uniform(m.n_cols * f, 2 + f, (m.n_cols, f))).cuda()

        def run():
            asb._check(_capi.lib.as_sddmm(C.byref(v), g.handle, C.c_void_p(x.data_ptr()), m.n_rows,
                                          C.c_void_p(y.data_ptr()), m.n_cols, f, C.c_void_p(out.data_ptr()),
                                          C.c_void_p(s), None))
        res, ref = {}, None
        for xp in ("0", "1", "2") * 3:
            os.environ["AUTOSAGE_DEV_SDDMM_XPOL"] = xp
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
            res.setdefault(xp, []).append(sorted(ts)[len(ts) // 2])
            if ref is None:
                ref = out.clone()
            assert torch.equal(ref.view(torch.int32), out.view(torch.int32)), (f, xp)
        print(f"F={f}: " + "  ".join(f"xpol={k} {min(t):.3f} ms" for k, t in res.items()), flush=True)
        del x, y


if __name__ == "__main__":
    main()
