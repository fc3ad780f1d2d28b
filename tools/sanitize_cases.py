#!/usr/bin/env python3
"""Small parity workload for compute-sanitizer (tests/test_sanitizer.py).

Runs every kernel family once on graphs small enough for the sanitizer's
instrumentation yet shaped to reach each code path, and checks the outputs
against the oracle (so a race that corrupts data also fails here):

  SpMM   lane-group kernel row mode (fast loop + ragged tail), hub pieces +
         reduce, the cp.async ring kernel (rows >= 256 on a small graph),
         baseline; f32, bf16 B, transpose values (backward)
  SDDMM  pair1 kernel (F=32, 64, 100), pair kernel (F=128), pass-major
         pair kernel (F=128, forced), chunk kernel (F=24), direct
         (baseline), bf16
  blocked SpMM (carried state, 3 column blocks, hub pieces)
  softmax warp / CTA / chain kernels, fused and staged attention

  python tools/sanitize_cases.py        # prints SANITIZE_CASES_OK
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
import paper_2511_17594_b200 as asb  # noqa: E402
import paper_2511_17594_b200.torch_ops  # noqa: E402,F401  (registers torch.ops.autosage)
from tests.util import bit_equal, csr_from_degrees, max_err, random_dense  # noqa: E402


def V(op, mapping, ft=64, rpc=1, vec=True, hubt=256):
    return asb.KernelVariant(op, mapping, ft, rpc, vec, hubt)


def main():
    rng = np.random.default_rng(2024)
    # 3 hubs (2 multi-piece), 40 rows of degree 256..600 (ring kernel), light rest
    deg = np.concatenate([[5000, 2300, 700], rng.integers(256, 600, 40), rng.integers(0, 48, 1957)])
    a = csr_from_degrees(rng, 2000, 6000, deg)
    g = asb.Graph.from_csr(a)
    for f in (32, 64, 100, 128):
        b = random_dense(rng, 6000, f)
        bd = torch.from_numpy(b).cuda()
        want = oracle.spmm_baseline(a, b)
        assert bit_equal(asb.spmm_baseline(g, bd).cpu().numpy(), want)
        for vec in (True, False):
            got = asb.dispatch(V(asb.SPMM, asb.ROWPARALLEL, 64, 4, vec), g, bd).output.cpu().numpy()
            assert bit_equal(got, want), ("rows", f, vec)
        got = asb.dispatch(V(asb.SPMM, asb.HUBSPLIT, 64, 1, True, 256), g, bd).output.cpu().numpy()
        assert bit_equal(got, oracle.spmm_hubsplit(a, b, 256)), ("hub", f)
        x = random_dense(rng, 2000, f)
        xd = torch.from_numpy(x).cuda()
        for ft, vec in ((32, False), (32, True)):
            got = asb.dispatch(V(asb.SDDMM, asb.ROWPARALLEL, ft, 1, vec), g, xd, bd).values.cpu().numpy()
            assert bit_equal(got, oracle.sddmm(a, x, b, ft, vec)), ("sddmm", f, ft, vec)
        assert bit_equal(asb.sddmm_baseline(g, xd, bd).cpu().numpy(), oracle.sddmm(a, x, b))
        if f in (32, 64):  # bf16 operands
            bb = bd.to(torch.bfloat16)
            got = torch.ops.autosage.spmm_csr(*_csr(a), bb, "spmm:hubsplit:ft=64:rpc=1:vec=1:hubt=256")
            assert bit_equal(got.cpu().numpy(), oracle.spmm_hubsplit(a, bb.float().cpu().numpy(), 256))
    # pass-major SDDMM (forced on this small graph) and the general chunk kernel
    for f, pm in ((128, "1"), (24, "0")):
        os.environ["AUTOSAGE_DEV_SDDMM_PM"] = pm
        x, y = random_dense(rng, 2000, f), random_dense(rng, 6000, f)
        xd, yd = torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda()
        for ft, vec in ((32, False), (32, True), (64, True)):
            got = asb.dispatch(V(asb.SDDMM, asb.ROWPARALLEL, ft, 1, vec), g, xd, yd).values.cpu().numpy()
            assert bit_equal(got, oracle.sddmm(a, x, y, ft, vec and f % 4 == 0)), ("sddmm pm", f, ft, vec)
    os.environ.pop("AUTOSAGE_DEV_SDDMM_PM", None)
    # column-blocked SpMM: carried f64 state across 3 blocks, hub pieces
    b = random_dense(rng, 6000, 64)
    bd = torch.from_numpy(b).cuda()
    cd = torch.empty((2000, 64), device="cuda")
    for var in (V(asb.SPMM, asb.HUBSPLIT, 64, 1, True, 256), None):
        bp = asb.BlockedSpmm(g, var, [0, 1500, 1501, 6000])
        for k in range(bp.n_blocks):
            bp.run(k, bd, cd)
        torch.cuda.synchronize()
        want = oracle.spmm_hubsplit(a, b, 256) if var is not None else oracle.spmm_baseline(a, b)
        assert bit_equal(cd.cpu().numpy(), want), ("blocked", var)
        bp.close()
    # softmax over wide scores (forces the chain path on long rows)
    vals = (rng.standard_normal(a.nnz) * 30).astype(np.float32)
    got = asb.row_softmax(a.with_values(vals)).val
    assert max_err(got, oracle.row_softmax(a, vals)) <= 1.0
    # attention: fused and staged
    q, k, v = (random_dense(rng, n, 64) for n in (2000, 6000, 6000))
    pat = asb.CsrMatrix(a.n_rows, a.n_cols, a.rowptr, a.colind, None)
    out_f = asb.csr_attention_forward(pat, q, k, v, fused=True)
    out_s = asb.csr_attention_forward(pat, q, k, v, fused=False)
    assert bit_equal(out_f, out_s)
    assert max_err(out_f, oracle.attention(pat, q, k, v)) <= 1.0
    # backward: transpose + values through the permutation
    crow, col, val = _csr(a)
    bt = torch.from_numpy(random_dense(rng, 6000, 32)).cuda().requires_grad_(True)
    c = torch.ops.autosage.spmm_csr(crow, col, val, bt, "")
    c.sum().backward()
    torch.cuda.synchronize()
    g.close()
    print("SANITIZE_CASES_OK")


def _csr(m):
    return (torch.from_numpy(m.rowptr.astype(np.int64)).cuda(), torch.from_numpy(m.colind.astype(np.int32)).cuda(),
            torch.from_numpy(m.val).cuda() if m.val is not None else torch.empty(0, device="cuda"))


if __name__ == "__main__":
    main()
