"""A/B the register budget (AUTOSAGE_DEV_SDDMM_BF16_MINB / _MINB) of the SDDMM
pair kernels on the Reddit-shape graph: python tools/tune_sddmm_bf16.py"""
import ctypes as C
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))

import torch  # noqa: E402

import bench  # noqa: E402
import paper_2511_17594_b200 as asb  # noqa: E402
from sweep import P, ev_time, lib  # noqa: E402


def main():
    m, _ = bench.make_graph("reddit", 1)
    g = asb.Graph.from_csr(m.with_values(None))
    dev = torch.device("cuda")
    stream = C.c_void_p(asb.torch_stream_handle())
    sd = asb.variant_from_string("sddmm:rowparallel:ft=32:rpc=1:vec=0:hubt=256").to_c()
    for f in (32, 64):
        x = torch.from_numpy(asb.fill_uniform(m.n_rows * f, 2 + f, (m.n_rows, f))).to(dev).to(torch.bfloat16)
        y = torch.from_numpy(asb.fill_uniform(m.n_cols * f, 3 + f, (m.n_cols, f))).to(dev).to(torch.bfloat16)
        out = torch.empty(m.nnz, dtype=torch.float32, device=dev)
        ref = None
        for minb in (3, 4, 5):
            os.environ["AUTOSAGE_DEV_SDDMM_BF16_MINB"] = str(minb)
            run = lambda: asb._check(lib.as_sddmm_bf16(C.byref(sd), g.handle, P(x), m.n_rows, P(y), m.n_cols, f,  # noqa: E731
                                                       P(out), stream, None))
            t = ev_time(run, 7, 2)
            o = out.clone()
            same = True if ref is None else bool(torch.equal(o.view(torch.int32), ref.view(torch.int32)))
            ref = o if ref is None else ref
            print(f"F={f} minb={minb}: {t:.3f} ms  same_bits={same}", flush=True)
    # f32 pair kernel at F=32 (AUTOSAGE_DEV_SDDMM_MINB)
    f = 32
    x = torch.from_numpy(asb.fill_uniform(m.n_rows * f, 2 + f, (m.n_rows, f))).to(dev)
    y = torch.from_numpy(asb.fill_uniform(m.n_cols * f, 3 + f, (m.n_cols, f))).to(dev)
    out = torch.empty(m.nnz, dtype=torch.float32, device=dev)
    ref = None
    for minb in (3, 4, 5):
        os.environ["AUTOSAGE_DEV_SDDMM_MINB"] = str(minb)
        run = lambda: asb._check(lib.as_sddmm(C.byref(sd), g.handle, P(x), m.n_rows, P(y), m.n_cols, f,  # noqa: E731
                                              P(out), stream, None))
        t = ev_time(run, 7, 2)
        o = out.clone()
        same = True if ref is None else bool(torch.equal(o.view(torch.int32), ref.view(torch.int32)))
        ref = o if ref is None else ref
        print(f"f32 F={f} minb={minb}: {t:.3f} ms  same_bits={same}", flush=True)


if __name__ == "__main__":
    main()
