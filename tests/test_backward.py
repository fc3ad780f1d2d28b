"""Backward pass (the reference has no gradients):
device CSR transpose, value permutation, SpMM with explicit values, the row
softmax gradient, and torch autograd through torch.ops.autosage.*.

Parity bar: structure and permutation bit-exact vs oracle.transpose; SpMM /
SDDMM gradients bit-exact vs the oracle's SpMM / SDDMM on the transposed or
re-valued CSR (they are the same kernels); softmax gradient bit-exact vs
oracle.row_softmax_backward (fixed summation order, oracle/oracle.c).
Float64 torch autograd on a dense copy checks the formulas themselves
(tolerance 1e-5 relative, the north-star value bar)."""
import numpy as np
import pytest
import torch

import oracle
import paper_2511_17594_b200 as asb
import paper_2511_17594_b200.torch_ops  # noqa: F401
from tests.util import bit_equal, csr_from_degrees, empty_rows, hub_graph, random_csr, random_dense


def _dense(m):
    d = np.zeros((m.n_rows, m.n_cols), dtype=np.float64)
    for i in range(m.n_rows):
        for e in range(int(m.rowptr[i]), int(m.rowptr[i + 1])):
            d[i, m.colind[e]] = m.val[e] if m.has_values() else 1.0
    return d


# ---------------------------------------------------------------- CPU: oracle

def test_oracle_transpose_matches_dense_and_is_canonical():
    rng = np.random.default_rng(3)
    m = random_csr(rng, 40, 55, 12)
    (rp, ci, val), perm = oracle.transpose(m)
    t = asb.CsrMatrix(m.n_cols, m.n_rows, rp, ci, val)
    assert asb.validate(t) is None
    assert np.array_equal(_dense(t), _dense(m).T)
    # perm maps every transposed entry to its source entry
    assert sorted(perm.tolist()) == list(range(m.nnz))
    assert np.array_equal(m.colind[perm], np.repeat(np.arange(m.n_cols), np.diff(rp.astype(np.int64))))
    # transpose of the transpose is the original
    (rp2, ci2, val2), _ = oracle.transpose(t)
    assert np.array_equal(rp2, m.rowptr) and np.array_equal(ci2, m.colind)
    assert bit_equal(val2, m.val)


def test_oracle_transpose_edge_cases():
    m = empty_rows(5, 7)
    (rp, ci, _), perm = oracle.transpose(m)
    assert rp.tolist() == [0] * 8 and ci.size == 0 and perm.size == 0
    m = asb.CsrMatrix(0, 3, np.zeros(1, dtype=np.uint64), np.zeros(0, dtype=np.uint32))
    (rp, _, _), _ = oracle.transpose(m)
    assert rp.tolist() == [0, 0, 0, 0]


def _softmax_bwd_py(m, p, g):
    """Pure-Python statement of the fixed order (256 strided partials, pairwise fold)."""
    out = np.zeros(m.nnz, dtype=np.float32)
    for i in range(m.n_rows):
        e0, e1 = int(m.rowptr[i]), int(m.rowptr[i + 1])
        part = [0.0] * 256
        for e in range(e0, e1):
            part[(e - e0) & 255] += float(p[e]) * float(g[e])
        o = 128
        while o:
            for l in range(o):
                part[l] += part[l + o]
            o >>= 1
        for e in range(e0, e1):
            out[e] = np.float32(float(p[e]) * (float(g[e]) - part[0]))
    return out


def test_oracle_softmax_backward_order_and_formula():
    rng = np.random.default_rng(4)
    m = csr_from_degrees(rng, 8, 1200, [0, 1, 31, 32, 33, 150, 256, 1100])
    s = rng.standard_normal(m.nnz).astype(np.float32) * 4
    p = oracle.row_softmax(m, s)
    g = rng.standard_normal(m.nnz).astype(np.float32)
    got = oracle.row_softmax_backward(m, p, g)
    assert bit_equal(got, _softmax_bwd_py(m, p, g))
    # the Jacobian-vector product of softmax, in f64 on a dense row
    for i in range(m.n_rows):
        e0, e1 = int(m.rowptr[i]), int(m.rowptr[i + 1])
        if e0 == e1:
            continue
        pp, gg = p[e0:e1].astype(np.float64), g[e0:e1].astype(np.float64)
        want = pp * (gg - (pp * gg).sum())
        assert np.allclose(got[e0:e1], want, rtol=1e-5, atol=1e-6)


def test_backward_ops_registered_with_fake_shapes():
    from torch._subclasses.fake_tensor import FakeTensorMode
    for name in ("row_softmax_csr", "row_softmax_csr_backward"):
        assert hasattr(torch.ops.autosage, name)
    with FakeTensorMode():
        crow = torch.empty(11, dtype=torch.int64)
        col = torch.empty(30, dtype=torch.int32)
        s = torch.empty(30)
        assert torch.ops.autosage.row_softmax_csr(crow, col, s, 7).shape == (30,)
        assert torch.ops.autosage.row_softmax_csr_backward(crow, col, s, s, 7).shape == (30,)
        # bf16 attention: float32 outputs of the f32 shapes
        q = torch.empty(10, 16, dtype=torch.bfloat16)
        kv = torch.empty(7, 8, dtype=torch.bfloat16)
        out = torch.ops.autosage.csr_attention(crow, col, q, torch.empty(7, 16, dtype=torch.bfloat16), kv, False)
        assert out.shape == (10, 8) and out.dtype == torch.float32
        out, p = torch.ops.autosage.csr_attention_with_probs(crow, col, q, torch.empty(7, 16, dtype=torch.bfloat16),
                                                            kv)
        assert out.dtype == p.dtype == torch.float32 and p.shape == (30,)


# ---------------------------------------------------------------- GPU: kernels

def _graphs():
    rng = np.random.default_rng(11)
    yield random_csr(rng, 300, 420, 25)
    yield hub_graph(rng, 1200, [1100, 700, 300], 9)
    yield csr_from_degrees(rng, 64, 5000, [0] * 10 + [4999] + [1] * 53)
    yield empty_rows(9, 4)


@pytest.mark.gpu
def test_device_transpose_bit_exact_vs_oracle():
    for m in _graphs():
        g = asb.Graph.from_csr(m)
        gt = g.transpose()
        t = gt.download()
        (rp, ci, val), perm = oracle.transpose(m)
        assert (gt.n_rows, gt.n_cols, gt.nnz) == (m.n_cols, m.n_rows, m.nnz)
        assert np.array_equal(t.rowptr, rp) and np.array_equal(t.colind, ci)
        if m.nnz:
            assert bit_equal(t.val, val)
            # the kept permutation, read through as_permute_values of iota (< 2^24: exact in f32)
            import ctypes as C
            from paper_2511_17594_b200 import _lib
            iota = torch.arange(m.nnz, dtype=torch.float32, device="cuda")
            out = torch.empty_like(iota)
            asb._check(_lib.as_permute_values(gt.handle, C.c_void_p(iota.data_ptr()),
                                              C.c_void_p(out.data_ptr()), None))
            torch.cuda.synchronize()
            assert np.array_equal(out.cpu().numpy().astype(np.uint32), perm)
            assert gt.transpose_perm_ptr() != 0
        gt.close()
        g.close()


@pytest.mark.gpu
def test_transpose_perm_rejects_non_transpose():
    m = random_csr(np.random.default_rng(1), 10, 10, 3)
    g = asb.Graph.from_csr(m)
    with pytest.raises(asb.InvalidArgument):
        g.transpose_perm_ptr()


@pytest.mark.gpu
def test_spmm_values_and_permute_match_oracle():
    import ctypes as C
    from paper_2511_17594_b200 import _lib
    rng = np.random.default_rng(12)
    m = hub_graph(rng, 1500, [1400, 500], 11)
    g = asb.Graph.from_csr(m.with_values(None))
    gt = g.transpose()
    (rp, ci, _), perm = oracle.transpose(m)
    w = rng.standard_normal(m.nnz).astype(np.float32)
    wd = torch.from_numpy(w).cuda()
    wt = torch.empty_like(wd)
    asb._check(_lib.as_permute_values(gt.handle, C.c_void_p(wd.data_ptr()), C.c_void_p(wt.data_ptr()), None))
    torch.cuda.synchronize()
    assert bit_equal(wt.cpu().numpy(), w[perm])
    for f in (1, 7, 64, 100):
        b = random_dense(rng, m.n_rows, f)
        bd = torch.from_numpy(b).cuda()
        c = torch.empty((m.n_cols, f), device="cuda")
        for v in (None, "spmm:rowparallel:ft=32:rpc=4:vec=1:hubt=256", "spmm:hubsplit:ft=64:rpc=1:vec=1:hubt=64"):
            va = None if v is None else C.byref(asb.variant_from_string(v).to_c())
            asb._check(_lib.as_spmm_values(va, gt.handle, C.c_void_p(wt.data_ptr()), C.c_void_p(bd.data_ptr()),
                                           m.n_rows, f, C.c_void_p(c.data_ptr()), None, None))
            torch.cuda.synchronize()
            want = oracle.spmm_baseline(asb.CsrMatrix(m.n_cols, m.n_rows, rp, ci, w[perm]), b)
            assert bit_equal(c.cpu().numpy(), want), (f, v)
    with pytest.raises(asb.InvalidArgument):
        asb._check(_lib.as_spmm_values(None, gt.handle, None, C.c_void_p(bd.data_ptr()), m.n_rows, f,
                                       C.c_void_p(c.data_ptr()), None, None))


@pytest.mark.gpu
def test_softmax_backward_bit_exact_vs_oracle():
    rng = np.random.default_rng(13)
    for m in (csr_from_degrees(rng, 10, 9000, [0, 1, 2, 31, 32, 33, 64, 2999, 4096, 8999]),
              hub_graph(rng, 6000, [5900, 4100, 1000], 40, with_values=False)):
        crow = torch.from_numpy(m.rowptr.astype(np.int64)).cuda()
        col = torch.from_numpy(m.colind.astype(np.int32)).cuda()
        s = (rng.standard_normal(m.nnz) * 5).astype(np.float32)
        p = oracle.row_softmax(m, s)
        gr = rng.standard_normal(m.nnz).astype(np.float32)
        got = torch.ops.autosage.row_softmax_csr_backward(crow, col, torch.from_numpy(p).cuda(),
                                                          torch.from_numpy(gr).cuda(), m.n_cols)
        assert bit_equal(got.cpu().numpy(), oracle.row_softmax_backward(m, p, gr))
        pd = torch.ops.autosage.row_softmax_csr(crow, col, torch.from_numpy(s).cuda(), m.n_cols)
        assert bit_equal(pd.cpu().numpy(), p)


# ---------------------------------------------------------------- GPU: autograd

def _t(a, grad=False):
    t = torch.from_numpy(np.ascontiguousarray(a)).cuda()
    return t.requires_grad_(grad)


@pytest.mark.gpu
def test_spmm_autograd_bit_exact_vs_oracle():
    rng = np.random.default_rng(21)
    m = hub_graph(rng, 900, [850, 400], 8)
    crow, col = _t(m.rowptr.astype(np.int64)), _t(m.colind.astype(np.int32))
    for f in (16, 64):
        b = random_dense(rng, m.n_cols, f)
        dc = random_dense(rng, m.n_rows, f)
        val, bt = _t(m.val, True), _t(b, True)
        for v in ("", "spmm:hubsplit:ft=32:rpc=4:vec=1:hubt=128"):
            val.grad = bt.grad = None
            out = torch.ops.autosage.spmm_csr(crow, col, val, bt, v)
            out.backward(_t(dc))
            (rp, ci, vt), perm = oracle.transpose(m)
            want_db = oracle.spmm_baseline(asb.CsrMatrix(m.n_cols, m.n_rows, rp, ci, vt), dc)
            want_dval = oracle.sddmm(m, dc, b)
            assert bit_equal(bt.grad.cpu().numpy(), want_db)
            assert bit_equal(val.grad.cpu().numpy(), want_dval)
    # formula check against dense f64 autograd
    bd = torch.from_numpy(b).double().requires_grad_(True)
    A = torch.from_numpy(_dense(m))
    (A @ bd).backward(torch.from_numpy(dc).double())
    assert np.allclose(bt.grad.cpu().numpy(), bd.grad.numpy(), rtol=1e-5, atol=1e-5)


@pytest.mark.gpu
def test_sddmm_autograd_bit_exact_vs_oracle():
    rng = np.random.default_rng(22)
    m = hub_graph(rng, 800, [790, 300], 10, with_values=False)
    crow, col = _t(m.rowptr.astype(np.int64)), _t(m.colind.astype(np.int32))
    x, y = random_dense(rng, m.n_rows, 32), random_dense(rng, m.n_cols, 32)
    dout = rng.standard_normal(m.nnz).astype(np.float32)
    xt, yt = _t(x, True), _t(y, True)
    torch.ops.autosage.sddmm_csr(crow, col, xt, yt, "").backward(_t(dout))
    want_dx = oracle.spmm_baseline(m.with_values(dout), y)
    (rp, ci, _), perm = oracle.transpose(m)
    want_dy = oracle.spmm_baseline(asb.CsrMatrix(m.n_cols, m.n_rows, rp, ci, dout[perm]), x)
    assert bit_equal(xt.grad.cpu().numpy(), want_dx)
    assert bit_equal(yt.grad.cpu().numpy(), want_dy)


@pytest.mark.gpu
def test_attention_autograd_matches_composed_oracle_and_f64():
    rng = np.random.default_rng(23)
    m = hub_graph(rng, 600, [590, 200], 7, with_values=False)
    crow, col = _t(m.rowptr.astype(np.int64)), _t(m.colind.astype(np.int32))
    q, k, v = (random_dense(rng, 600, 16) for _ in range(3))
    do = random_dense(rng, 600, 16)
    qt, kt, vt = _t(q, True), _t(k, True), _t(v, True)
    for fused in (False, True):
        qt.grad = kt.grad = vt.grad = None
        torch.ops.autosage.csr_attention(crow, col, qt, kt, vt, fused).backward(_t(do))
        # composed oracle: the same staged recompute
        s = oracle.sddmm(m, q, k)
        p = oracle.row_softmax(m, s)
        (rp, ci, _), perm = oracle.transpose(m)
        mt = lambda w: asb.CsrMatrix(m.n_cols, m.n_rows, rp, ci, w[perm])  # noqa: E731
        want_dv = oracle.spmm_baseline(mt(p), do)
        dp = oracle.sddmm(m, do, v)
        ds = oracle.row_softmax_backward(m, p, dp)
        want_dq = oracle.spmm_baseline(m.with_values(ds), k)
        want_dk = oracle.spmm_baseline(mt(ds), q)
        assert bit_equal(vt.grad.cpu().numpy(), want_dv)
        assert bit_equal(qt.grad.cpu().numpy(), want_dq)
        assert bit_equal(kt.grad.cpu().numpy(), want_dk)
    # formulas vs dense f64 autograd (masked softmax attention)
    mask = torch.from_numpy(_dense(m) != 0)
    Q, K, V = (torch.from_numpy(a).double().requires_grad_(True) for a in (q, k, v))
    S = (Q @ K.T).masked_fill(~mask, float("-inf"))
    P = torch.softmax(S, dim=1).nan_to_num(0.0)
    (P @ V).backward(torch.from_numpy(do).double())
    for got, want in ((qt, Q), (kt, K), (vt, V)):
        assert np.allclose(got.grad.cpu().numpy(), want.grad.numpy(), rtol=1e-4, atol=1e-5)


# ---------------------------------------------------------------- GPU: bf16 B

def _bf16_words(rng, rows, f):
    """bf16 bit patterns of U(-1,1) values, and their exact f32 values."""
    x = (rng.random((rows, f), dtype=np.float32) * 2 - 1).astype(np.float32)
    w = (x.view(np.uint32) >> 16).astype(np.uint16)
    return w, (w.astype(np.uint32) << 16).view(np.float32)


@pytest.mark.gpu
def test_spmm_bf16_bit_exact_vs_oracle_on_widened_b():
    import ctypes as C
    from paper_2511_17594_b200 import _lib
    rng = np.random.default_rng(31)
    for m in (hub_graph(rng, 1300, [1250, 600, 300], 9), hub_graph(rng, 700, [650], 5, with_values=False)):
        g = asb.Graph.from_csr(m)
        for f in (1, 6, 16, 64, 100, 132, 512):
            w, bf = _bf16_words(rng, m.n_cols, f)
            if f == 16:
                w[3, 2] = 0x7F80     # +Inf: the finite scan must route to the F2F widening
                bf = (w.astype(np.uint32) << 16).view(np.float32)
            wd = torch.from_numpy(w.view(np.int16)).cuda()
            c = torch.empty((m.n_rows, f), device="cuda")
            want = oracle.spmm_baseline(m, bf)
            for v in (None, "spmm:rowparallel:ft=64:rpc=4:vec=1:hubt=256", "spmm:rowparallel:ft=32:rpc=1:vec=0:hubt=256",
                      "spmm:hubsplit:ft=64:rpc=1:vec=1:hubt=64", "spmm:hubsplit:ft=128:rpc=4:vec=1:hubt=400",
                      "spmm:rowparallel:ft=1024:rpc=4:vec=1:hubt=256"):
                va = None if v is None else C.byref(asb.variant_from_string(v).to_c())
                res = asb._capi.as_kernel_result()
                asb._check(_lib.as_spmm_bf16(va, g.handle, None, C.c_void_p(wd.data_ptr()), m.n_cols, f,
                                             C.c_void_p(c.data_ptr()), None, C.byref(res)))
                torch.cuda.synchronize()
                got = c.cpu().numpy()
                if v is not None and "hubsplit" in v:
                    hubt = int(v.rsplit("=", 1)[1])
                    ref = oracle.spmm_hubsplit(m, bf, hubt)
                else:
                    ref = want
                assert bit_equal(got, ref), (f, v)
        # misaligned base (2-byte offset): the scalar path
        w, bf = _bf16_words(rng, m.n_cols + 1, 8)
        wd = torch.from_numpy(w.view(np.int16).reshape(-1)).cuda()
        c = torch.empty((m.n_rows, 8), device="cuda")
        va = C.byref(asb.variant_from_string("spmm:rowparallel:ft=64:rpc=4:vec=1:hubt=256").to_c())
        asb._check(_lib.as_spmm_bf16(va, g.handle, None, C.c_void_p(wd.data_ptr() + 2), m.n_cols, 8,
                                     C.c_void_p(c.data_ptr()), None, None))
        torch.cuda.synchronize()
        shifted = bf.reshape(-1)[1:1 + m.n_cols * 8].reshape(m.n_cols, 8)
        assert bit_equal(c.cpu().numpy(), oracle.spmm_baseline(m, shifted))
        g.close()


@pytest.mark.gpu
def test_spmm_op_bf16_forward_and_grad():
    rng = np.random.default_rng(32)
    m = hub_graph(rng, 600, [560], 6)
    crow, col = _t(m.rowptr.astype(np.int64)), _t(m.colind.astype(np.int32))
    w, bf = _bf16_words(rng, m.n_cols, 64)
    b16 = torch.from_numpy(w.view(np.int16)).cuda().view(torch.bfloat16).requires_grad_(True)
    out = torch.ops.autosage.spmm_csr(crow, col, _t(m.val), b16, "spmm:hubsplit:ft=64:rpc=1:vec=1:hubt=256")
    assert out.dtype == torch.float32
    assert bit_equal(out.detach().cpu().numpy(), oracle.spmm_hubsplit(m, bf, 256))
    out.sum().backward()
    assert b16.grad.dtype == torch.bfloat16


@pytest.mark.gpu
def test_sddmm_bf16_bit_exact_vs_oracle_on_widened_operands():
    import ctypes as C
    from paper_2511_17594_b200 import _lib
    rng = np.random.default_rng(33)
    for m in (hub_graph(rng, 1100, [1000, 400], 9, with_values=False), random_csr(rng, 500, 700, 40)):
        g = asb.Graph.from_csr(m.with_values(None))
        for f in (1, 12, 32, 64, 80):
            wx, bx = _bf16_words(rng, m.n_rows, f)
            wy, by = _bf16_words(rng, m.n_cols, f)
            if f == 64:
                wy[5, 7] = 0x7FC0    # NaN in Y: the F2F widening path, NaN propagates
                by = (wy.astype(np.uint32) << 16).view(np.float32)
            xd = torch.from_numpy(wx.view(np.int16)).cuda()
            yd = torch.from_numpy(wy.view(np.int16)).cuda()
            out = torch.empty(max(m.nnz, 1), device="cuda")
            for v in (None, "sddmm:rowparallel:ft=32:rpc=1:vec=0:hubt=256", "sddmm:rowparallel:ft=32:rpc=4:vec=1:hubt=256",
                      "sddmm:hubsplit:ft=64:rpc=4:vec=1:hubt=256", "sddmm:rowparallel:ft=128:rpc=1:vec=1:hubt=256"):
                va = None if v is None else C.byref(asb.variant_from_string(v).to_c())
                asb._check(_lib.as_sddmm_bf16(va, g.handle, C.c_void_p(xd.data_ptr()), m.n_rows,
                                              C.c_void_p(yd.data_ptr()), m.n_cols, f, C.c_void_p(out.data_ptr()),
                                              None, None))
                torch.cuda.synchronize()
                if v is None:
                    want = oracle.sddmm(m, bx, by, f, False)
                else:
                    var = asb.variant_from_string(v)
                    want = oracle.sddmm(m, bx, by, var.f_tile, var.vectorized and f % 4 == 0)
                got = out.cpu().numpy()[:m.nnz]
                nan = np.isnan(want)
                assert np.array_equal(np.isnan(got), nan), (f, v)   # NaN payloads are not compared
                assert bit_equal(got[~nan], want[~nan]), (f, v)
        g.close()


@pytest.mark.gpu
def test_sddmm_op_bf16_forward_and_grad():
    rng = np.random.default_rng(34)
    m = hub_graph(rng, 400, [380], 6, with_values=False)
    crow, col = _t(m.rowptr.astype(np.int64)), _t(m.colind.astype(np.int32))
    wx, bx = _bf16_words(rng, m.n_rows, 64)
    wy, by = _bf16_words(rng, m.n_cols, 64)
    x16 = torch.from_numpy(wx.view(np.int16)).cuda().view(torch.bfloat16).requires_grad_(True)
    y16 = torch.from_numpy(wy.view(np.int16)).cuda().view(torch.bfloat16).requires_grad_(True)
    out = torch.ops.autosage.sddmm_csr(crow, col, x16, y16, "sddmm:rowparallel:ft=32:rpc=1:vec=0:hubt=256")
    assert out.dtype == torch.float32
    assert bit_equal(out.detach().cpu().numpy(), oracle.sddmm(m, bx, by, 32, False))
    out.sum().backward()
    assert x16.grad.dtype == torch.bfloat16 and y16.grad.dtype == torch.bfloat16


@pytest.mark.gpu
@pytest.mark.parametrize("merged", ["1", "2"])
def test_spmm_transpose_values_equals_permute_then_spmm(monkeypatch, merged):
    """A^T products with the values loaded through the entry permutation; with
    AUTOSAGE_DEV_SPMM_MERGED=2 the hub-split runs as one launch over pieces +
    light rows even on these small graphs."""
    import ctypes as C
    from paper_2511_17594_b200 import _lib
    monkeypatch.setenv("AUTOSAGE_DEV_SPMM_MERGED", merged)
    rng = np.random.default_rng(35)
    for m in (hub_graph(rng, 1500, [1400, 500], 11), random_csr(rng, 300, 300, 30)):
        g = asb.Graph.from_csr(m.with_values(None))
        gt = g.transpose()
        (rp, ci, _), perm = oracle.transpose(m)
        w = rng.standard_normal(m.nnz).astype(np.float32)
        wd = torch.from_numpy(w).cuda()
        for f in (3, 64, 100):
            b = random_dense(rng, m.n_rows, f)
            bd = torch.from_numpy(b).cuda()
            c = torch.empty((m.n_cols, f), device="cuda")
            want = oracle.spmm_baseline(asb.CsrMatrix(m.n_cols, m.n_rows, rp, ci, w[perm]), b)
            for v in (None, "spmm:rowparallel:ft=64:rpc=4:vec=1:hubt=256", "spmm:hubsplit:ft=32:rpc=1:vec=0:hubt=64",
                      "spmm:hubsplit:ft=64:rpc=1:vec=1:hubt=256"):
                va = None if v is None else C.byref(asb.variant_from_string(v).to_c())
                asb._check(_lib.as_spmm_transpose_values(va, gt.handle, C.c_void_p(wd.data_ptr()),
                                                         C.c_void_p(bd.data_ptr()), m.n_rows, f,
                                                         C.c_void_p(c.data_ptr()), None, None))
                torch.cuda.synchronize()
                assert bit_equal(c.cpu().numpy(), want), (f, v)
        with pytest.raises(asb.InvalidArgument):
            asb._check(_lib.as_spmm_transpose_values(None, g.handle, C.c_void_p(wd.data_ptr()),
                                                     C.c_void_p(bd.data_ptr()), m.n_cols, f,
                                                     C.c_void_p(c.data_ptr()), None, None))
        gt.close()
        g.close()


@pytest.mark.gpu
def test_attention_with_probs_forward_and_grads_match_recompute_path():
    from paper_2511_17594_b200.torch_ops import csr_attention_train
    rng = np.random.default_rng(36)
    m = hub_graph(rng, 700, [650, 300], 7, with_values=False)
    crow, col = _t(m.rowptr.astype(np.int64)), _t(m.colind.astype(np.int32))
    q, k, v = (random_dense(rng, 700, 32) for _ in range(3))
    do = random_dense(rng, 700, 32)
    grads = []
    for fn in (lambda a, b, c: torch.ops.autosage.csr_attention(crow, col, a, b, c, True),
               lambda a, b, c: csr_attention_train(crow, col, a, b, c)):
        qt, kt, vt = _t(q, True), _t(k, True), _t(v, True)
        out = fn(qt, kt, vt)
        out.backward(_t(do))
        grads.append((out.detach().cpu().numpy(), qt.grad.cpu().numpy(), kt.grad.cpu().numpy(),
                      vt.grad.cpu().numpy()))
    for a, b in zip(*grads):
        assert bit_equal(a, b)
    out, p = torch.ops.autosage.csr_attention_with_probs(crow, col, _t(q), _t(k), _t(v))
    assert bit_equal(p.cpu().numpy(), oracle.row_softmax(m, oracle.sddmm(m, q, k)))


@pytest.mark.gpu
def test_attention_bf16_bit_exact_vs_oracle_on_widened_operands():
    """bf16 q, k, v: (out, p) equal the oracle's staged attention on the
    widened f32 operands (sequential SDDMM order, hub-split SpMM at hubT 256),
    bit for bit; grads come back in bf16 and match the f32 op's on the
    widened operands."""
    from paper_2511_17594_b200.torch_ops import csr_attention_train
    rng = np.random.default_rng(37)
    for m, f in ((hub_graph(rng, 900, [880, 400], 9, with_values=False), 64),
                 (random_csr(rng, 300, 300, 20).with_values(None), 32),
                 (empty_rows(9, 4).with_values(None), 16)):
        crow, col = _t(m.rowptr.astype(np.int64)), _t(m.colind.astype(np.int32))
        (wq, bq), (wk, bk), (wv, bv) = (_bf16_words(rng, m.n_rows, f) for _ in range(3))
        b16 = lambda w: torch.from_numpy(w.view(np.int16)).cuda().view(torch.bfloat16)  # noqa: E731
        want_p = oracle.row_softmax(m, oracle.sddmm(m, bq, bk, 32, False))
        want = oracle.attention(m, bq, bk, bv, 32, False, 256)
        out = torch.ops.autosage.csr_attention(crow, col, b16(wq), b16(wk), b16(wv), True)
        assert out.dtype == torch.float32
        assert bit_equal(out.cpu().numpy(), want)
        out, p = torch.ops.autosage.csr_attention_with_probs(crow, col, b16(wq), b16(wk), b16(wv))
        assert bit_equal(p.cpu().numpy(), want_p)
        assert bit_equal(out.cpu().numpy(), want)
        if m.nnz == 0:
            continue
        do = _t(random_dense(rng, m.n_rows, f))
        q16, k16, v16 = (b16(w).requires_grad_(True) for w in (wq, wk, wv))
        csr_attention_train(crow, col, q16, k16, v16).backward(do)
        qf, kf, vf = (_t(a, True) for a in (bq, bk, bv))
        torch.ops.autosage.csr_attention(crow, col, qf, kf, vf, False).backward(do)
        for g16, gf in ((q16, qf), (k16, kf), (v16, vf)):
            assert g16.grad.dtype == torch.bfloat16
            assert torch.equal(g16.grad, gf.grad.to(torch.bfloat16))
