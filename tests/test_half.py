"""16-bit dense operands: bf16 and IEEE f16
words, read as such by the gather kernels (csrc/half.cuh), widen to f32
exactly, so every result must equal the f32 path on the widened operands bit
for bit -- SpMM (every mapping, 1-/4-/8-wide tiles, Inf gating the re-bias
widening, f16 subnormals), SDDMM (both orders, NaN), and CSR attention on
16-bit q, k, v, fused (probabilities applied inside the SpMM) and staged."""
import ctypes as C

import numpy as np
import pytest
import torch

import oracle
import paper_2511_17594_b200 as asb
import paper_2511_17594_b200.torch_ops  # noqa: F401
from paper_2511_17594_b200 import _lib
from tests.util import bit_equal, hub_graph, random_csr, random_dense

DTYPES = ["bf16", "f16"]


def words(rng, rows, f, kind):
    """16-bit patterns of U(-1,1) values (f16: with subnormals mixed in) and
    their exact f32 values."""
    x = (rng.random((rows, f), dtype=np.float32) * 2 - 1).astype(np.float32)
    if kind == "bf16":
        w = (x.view(np.uint32) >> 16).astype(np.uint16)
        return w, (w.astype(np.uint32) << 16).view(np.float32)
    if x.size > 8:
        x.reshape(-1)[::97] *= 1e-6  # f16 subnormals (< 6.1e-5)
    h = x.astype(np.float16)
    return h.view(np.uint16), h.astype(np.float32)


def widen(w, kind):
    if kind == "bf16":
        return (w.astype(np.uint32) << 16).view(np.float32)
    return w.view(np.float16).astype(np.float32)


INF = {"bf16": 0x7F80, "f16": 0x7C00}
NAN = {"bf16": 0x7FC0, "f16": 0x7E00}
TORCH = {"bf16": torch.bfloat16, "f16": torch.float16}


def spmm_fn(kind):
    return _lib.as_spmm_bf16 if kind == "bf16" else _lib.as_spmm_f16


def sddmm_fn(kind):
    return _lib.as_sddmm_bf16 if kind == "bf16" else _lib.as_sddmm_f16


def t(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


@pytest.mark.gpu
@pytest.mark.parametrize("kind", DTYPES)
def test_spmm_half_bit_exact_on_widened_b(kind):
    rng = np.random.default_rng(131)
    for m in (hub_graph(rng, 1300, [1250, 600, 300], 9), hub_graph(rng, 700, [650], 5, with_values=False)):
        g = asb.Graph.from_csr(m)
        for f in (1, 6, 16, 64, 100, 132, 512):
            w, bf = words(rng, m.n_cols, f, kind)
            if f == 16:
                w[3, 2] = INF[kind]  # +Inf: the finite scan routes to the F2F widening
                bf = widen(w, kind)
            wd = torch.from_numpy(w.view(np.int16)).cuda()
            c = torch.empty((m.n_rows, f), device="cuda")
            for v in (None, "spmm:rowparallel:ft=64:rpc=4:vec=1:hubt=256", "spmm:rowparallel:ft=32:rpc=1:vec=0:hubt=256",
                      "spmm:hubsplit:ft=64:rpc=1:vec=1:hubt=64", "spmm:hubsplit:ft=128:rpc=4:vec=1:hubt=400"):
                va = None if v is None else C.byref(asb.variant_from_string(v).to_c())
                asb._check(spmm_fn(kind)(va, g.handle, None, C.c_void_p(wd.data_ptr()), m.n_cols, f,
                                         C.c_void_p(c.data_ptr()), None, None))
                torch.cuda.synchronize()
                ref = (oracle.spmm_hubsplit(m, bf, int(v.rsplit("=", 1)[1])) if v and "hubsplit" in v
                       else oracle.spmm_baseline(m, bf))
                assert bit_equal(c.cpu().numpy(), ref), (kind, f, v)
        g.close()


@pytest.mark.gpu
@pytest.mark.parametrize("kind", DTYPES)
def test_sddmm_half_bit_exact_on_widened_operands(kind):
    rng = np.random.default_rng(133)
    for m in (hub_graph(rng, 1100, [1000, 400], 9, with_values=False), random_csr(rng, 500, 700, 40)):
        g = asb.Graph.from_csr(m.with_values(None))
        for f in (1, 12, 32, 64, 80):
            wx, bx = words(rng, m.n_rows, f, kind)
            wy, by = words(rng, m.n_cols, f, kind)
            if f == 64:
                wy[5, 7] = NAN[kind]  # NaN in Y: the F2F path, NaN propagates
                by = widen(wy, kind)
            xd, yd = (torch.from_numpy(w.view(np.int16)).cuda() for w in (wx, wy))
            out = torch.empty(max(m.nnz, 1), device="cuda")
            for v in (None, "sddmm:rowparallel:ft=32:rpc=1:vec=0:hubt=256", "sddmm:rowparallel:ft=32:rpc=4:vec=1:hubt=256",
                      "sddmm:hubsplit:ft=64:rpc=4:vec=1:hubt=256"):
                va = None if v is None else C.byref(asb.variant_from_string(v).to_c())
                asb._check(sddmm_fn(kind)(va, g.handle, C.c_void_p(xd.data_ptr()), m.n_rows, C.c_void_p(yd.data_ptr()),
                                          m.n_cols, f, C.c_void_p(out.data_ptr()), None, None))
                torch.cuda.synchronize()
                if v is None:
                    want = oracle.sddmm(m, bx, by, f, False)
                else:
                    var = asb.variant_from_string(v)
                    want = oracle.sddmm(m, bx, by, var.f_tile, var.vectorized and f % 4 == 0)
                got = out.cpu().numpy()[:m.nnz]
                nan = np.isnan(want)
                assert np.array_equal(np.isnan(got), nan), (kind, f, v)
                assert bit_equal(got[~nan], want[~nan]), (kind, f, v)
        g.close()


@pytest.mark.gpu
@pytest.mark.parametrize("kind", DTYPES)
def test_attention_half_fused_and_staged(kind):
    """16-bit q, k, v: fused (scores -> row (max, sum) -> SpMM applying the
    softmax as it loads each score) and staged forms both equal the oracle's
    staged attention on the widened operands (sequential SDDMM, hub-split
    SpMM at hubT 256), bit for bit; p equals the oracle's probabilities."""
    rng = np.random.default_rng(137)
    for m, f in ((hub_graph(rng, 900, [880, 400], 9, with_values=False), 64),
                 (random_csr(rng, 300, 300, 20).with_values(None), 32),
                 (hub_graph(rng, 600, [500], 7, with_values=False), 128)):
        crow, col = t(m.rowptr.astype(np.int64)), t(m.colind.astype(np.int32))
        (wq, bq), (wk, bk), (wv, bv) = (words(rng, n, f, kind) for n in (m.n_rows, m.n_cols, m.n_cols))
        h = lambda w: torch.from_numpy(w.view(np.int16)).cuda().view(TORCH[kind])  # noqa: E731
        want = oracle.attention(m, bq, bk, bv, 32, False, 256)
        want_p = oracle.row_softmax(m, oracle.sddmm(m, bq, bk, 32, False))
        fused = torch.ops.autosage.csr_attention(crow, col, h(wq), h(wk), h(wv), True)
        staged = torch.ops.autosage.csr_attention(crow, col, h(wq), h(wk), h(wv), False)
        assert bit_equal(fused.cpu().numpy(), want) and bit_equal(staged.cpu().numpy(), want), (kind, f)
        out, p = torch.ops.autosage.csr_attention_with_probs(crow, col, h(wq), h(wk), h(wv))
        assert bit_equal(out.cpu().numpy(), want) and bit_equal(p.cpu().numpy(), want_p), (kind, f)


@pytest.mark.gpu
@pytest.mark.parametrize("kind", DTYPES)
def test_half_torch_ops_forward_and_grad(kind):
    rng = np.random.default_rng(139)
    m = hub_graph(rng, 600, [560], 6)
    crow, col = t(m.rowptr.astype(np.int64)), t(m.colind.astype(np.int32))
    w, bf = words(rng, m.n_cols, 64, kind)
    b16 = torch.from_numpy(w.view(np.int16)).cuda().view(TORCH[kind]).requires_grad_(True)
    out = torch.ops.autosage.spmm_csr(crow, col, t(m.val), b16, "spmm:hubsplit:ft=64:rpc=1:vec=1:hubt=256")
    assert out.dtype == torch.float32
    assert bit_equal(out.detach().cpu().numpy(), oracle.spmm_hubsplit(m, bf, 256))
    out.sum().backward()
    assert b16.grad.dtype == TORCH[kind]
    wx, bx = words(rng, m.n_rows, 32, kind)
    wy, by = words(rng, m.n_cols, 32, kind)
    x16, y16 = (torch.from_numpy(w_.view(np.int16)).cuda().view(TORCH[kind]) for w_ in (wx, wy))
    s = torch.ops.autosage.sddmm_csr(crow, col, x16, y16, "sddmm:rowparallel:ft=32:rpc=1:vec=0:hubt=256")
    assert bit_equal(s.cpu().numpy(), oracle.sddmm(m, bx, by, 32, False))
