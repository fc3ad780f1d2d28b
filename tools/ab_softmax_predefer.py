#!/usr/bin/env python3
"""Early chain deferral in the softmax CTA kernel (AUTOSAGE_DEV_SOFTMAX_PREDEFER
0 / 1): Reddit-shape fused attention (F=64, one head; q, k, v U(-1,1)) and a
row softmax over wide-range values, L2 flushed before each call, same bits
required.
  python tools/ab_softmax_predefer.py"""
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
    m, _ = bench.make_graph("reddit", 1)
    crow = torch.from_numpy(m.rowptr.astype(np.int64)).cuda()
    col = torch.from_numpy(m.colind.astype(np.int32)).cuda()
    f = 64
    q = torch.from_numpy(asb.fill_uniform(m.n_rows * f, 11, (m.n_rows, f))).cuda()
    k = torch.from_numpy(asb.fill_uniform(m.n_cols * f, 12, (m.n_cols, f))).cuda()
    v = torch.from_numpy(asb.fill_uniform(m.n_cols * f, 13, (m.n_cols, f))).cuda()
    flush = torch.empty(64 << 20, device="cuda")
    wide = torch.from_numpy((np.random.default_rng(5).standard_normal(m.nnz) * 8).astype(np.float32)).cuda()

    def att():
        return torch.ops.autosage.csr_attention(crow, col, q, k, v, True)

    def smx():
        return torch.ops.autosage.row_softmax_csr(crow, col, wide, m.n_cols)
    for name, fn in (("attention fused F=64", att), ("row_softmax sd=8", smx)):
        res, ref = {}, None
        for knob in ("0", "1", "2") * 3:
            os.environ["AUTOSAGE_DEV_SOFTMAX_PREDEFER"] = knob
            out = fn()
            torch.cuda.synchronize()
            evs = []
            for _ in range(5):
                flush.zero_()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                out = fn()
                e1.record()
                evs.append((e0, e1))
            torch.cuda.synchronize()
            ts = sorted(a.elapsed_time(b) for a, b in evs)
            res.setdefault(knob, []).append(ts[2])
            if ref is None:
                ref = out.clone()
            assert torch.equal(ref.view(torch.int32), out.view(torch.int32)), (name, knob)
        print(f"{name}: " + "  ".join(f"predefer={k} {min(t):.3f} ms" for k, t in res.items()) + "  bit-identical", flush=True)


if __name__ == "__main__":
    main()
