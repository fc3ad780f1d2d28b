"""Degenerate shapes through every operator family (the reference's own
edge cases, proj/tests/test_kernels.cpp:72-81, :178-187, plus the ones its
API admits but never tests): graphs with no rows, rows with no entries,
F = 0 and F = 1, a single entry, a hub threshold of 1 (one-entry pieces),
zero-column dense operands -- on the host-buffer path, the device path, the
scheduler (decide on an empty graph), attention, the column-blocked SpMM
and the 16-bit operand ops.  Results must equal the oracle (zeros of the
right shape, +0.0, and no launch error)."""
import ctypes as C

import numpy as np
import pytest
import torch

import oracle
import paper_2511_17594_b200 as asb
import paper_2511_17594_b200.torch_ops  # noqa: F401
from tests.util import bit_equal, random_dense

pytestmark = pytest.mark.gpu

SP, SD = asb.SPMM, asb.SDDMM
RP, HS = asb.ROWPARALLEL, asb.HUBSPLIT


def V(op, mapping, ft=64, rpc=1, vec=True, hubt=256):
    return asb.KernelVariant(op, mapping, ft, rpc, vec, hubt)


def csr(n_rows, n_cols, rowptr, colind, val=None):
    return asb.CsrMatrix(n_rows, n_cols, np.asarray(rowptr, np.uint64), np.asarray(colind, np.uint32),
                         None if val is None else np.asarray(val, np.float32))


def shapes():
    rng = np.random.default_rng(71)
    one = csr(1, 1, [0, 1], [0], [2.5])
    return [
        ("no rows", csr(0, 5, [0], [])),
        ("no entries", csr(3, 4, [0, 0, 0, 0], [])),
        ("no entries, no columns", csr(2, 0, [0, 0, 0], [])),
        ("single entry", one),
        ("last row only", csr(4, 3, [0, 0, 0, 0, 2], [0, 2], [1.5, -2.0])),
        ("ragged", csr(5, 6, [0, 3, 3, 4, 4, 6], [0, 2, 5, 1, 0, 5], rng.uniform(-1, 1, 6))),
    ]


@pytest.mark.parametrize("f", [0, 1, 5, 64])
def test_spmm_degenerate_every_mapping(f):
    rng = np.random.default_rng(72 + f)
    for name, m in shapes():
        b = random_dense(rng, m.n_cols, f)
        want = oracle.spmm_baseline(m, b) if m.n_rows and f else np.zeros((m.n_rows, f), np.float32)
        got = asb.spmm_baseline(m, b)
        assert got.shape == (m.n_rows, f) and bit_equal(got, want), (name, f)
        for v in (V(SP, RP, 64, 4, True), V(SP, RP, 1, 1, False), V(SP, HS, 64, 1, True, 1),
                  V(SP, HS, 32, 1, False, 256)):
            got = asb.dispatch(v, m, b).output
            assert got.shape == (m.n_rows, f), (name, f, v)
            assert bit_equal(got, want) and not np.any(np.signbit(got[want == 0])), (name, f, v)
        if m.n_rows:  # device operands
            g = asb.Graph.from_csr(m)
            bd = torch.from_numpy(b).cuda()
            got = asb.dispatch(V(SP, HS, 64, 1, True, 1), g, bd).output
            torch.cuda.synchronize()
            assert bit_equal(got.cpu().numpy(), want), (name, f, "device")
            g.close()


@pytest.mark.parametrize("f", [0, 1, 4, 64])
def test_sddmm_degenerate_both_orders(f):
    rng = np.random.default_rng(82 + f)
    for name, m in shapes():
        p = m.with_values(None)
        x, y = random_dense(rng, m.n_rows, f), random_dense(rng, m.n_cols, f)
        want_seq = oracle.sddmm(p, x, y) if m.nnz else np.zeros(0, np.float32)
        got = asb.sddmm_baseline(p, x, y)
        assert got.shape == (m.nnz,) and bit_equal(got, want_seq), (name, f)
        if f == 0 and m.nnz:
            assert np.all(got == 0.0) and not np.any(np.signbit(got))
        for vec in (False, True):
            got = asb.dispatch(V(SD, RP, 32, 1, vec), p, x, y).values
            want = oracle.sddmm(p, x, y, 32, vec and f % 4 == 0 and f > 0) if m.nnz else want_seq
            assert got.shape == (m.nnz,) and bit_equal(got, want), (name, f, vec)


def test_row_softmax_and_attention_degenerate():
    rng = np.random.default_rng(91)
    for name, m in shapes():
        vals = rng.uniform(-3, 3, m.nnz).astype(np.float32)
        got = asb.row_softmax(m.with_values(vals))
        assert got.nnz == m.nnz
        if m.nnz:
            assert np.array_equal(got.val, oracle.row_softmax(m, vals)) or \
                np.max(np.abs(got.val - oracle.row_softmax(m, vals))) <= 1e-6, name
        pat = m.with_values(None)
        q, k, v = random_dense(rng, m.n_rows, 8), random_dense(rng, m.n_cols, 8), random_dense(rng, m.n_cols, 8)
        for fused in (True, False):
            out = asb.csr_attention_forward(pat, q, k, v, fused=fused)
            assert out.shape == (m.n_rows, 8), (name, fused)
            if m.nnz:
                want = oracle.attention(pat, q, k, v)
                assert np.max(np.abs(out - want) - (1e-6 + 1e-5 * np.abs(want))) <= 0, (name, fused)
            else:
                assert np.all(out == 0.0), (name, fused)


def test_scheduler_decides_on_degenerate_graphs():
    """decide + auto on graphs with no entries (the reference probes the
    baseline and the shortlist even there; the result must be zeros)."""
    rng = np.random.default_rng(93)
    for name, m in shapes():
        for f in (1, 16):
            b = random_dense(rng, m.n_cols, f)
            cache = asb.ScheduleCache()
            ctx = asb.ScheduleContext(cache=cache)
            c = asb.spmm_auto(m, b, ctx=ctx)
            c = c[0] if isinstance(c, tuple) else c
            c = c.output if hasattr(c, "output") else c
            want = oracle.spmm_baseline(m, b) if m.n_rows else np.zeros((0, f), np.float32)
            assert np.asarray(c).shape == (m.n_rows, f) and bit_equal(np.asarray(c), want), (name, f)
            x, y = random_dense(rng, m.n_rows, f), random_dense(rng, m.n_cols, f)
            s = asb.sddmm_auto(m.with_values(None), x, y, ctx=ctx)
            s = s[0] if isinstance(s, tuple) else s
            s = s.values if hasattr(s, "values") else s
            assert np.asarray(s).shape == (m.nnz,), (name, f)
            if m.nnz:
                assert bit_equal(np.asarray(s), oracle.sddmm(m.with_values(None), x, y)) or \
                    bit_equal(np.asarray(s), oracle.sddmm(m.with_values(None), x, y, 32, f % 4 == 0)), (name, f)


def test_blocked_spmm_degenerate():
    rng = np.random.default_rng(95)
    for name, m in shapes():
        if m.n_rows == 0:
            continue
        g = asb.Graph.from_csr(m)
        f = 4
        b = torch.from_numpy(random_dense(rng, m.n_cols, f)).cuda()
        c = torch.full((m.n_rows, f), 7.0, device="cuda")
        cuts = [0, m.n_cols] if m.n_cols < 2 else [0, m.n_cols // 2, m.n_cols // 2, m.n_cols]
        for var in (None, V(SP, HS, 64, 1, True, 1)):
            bp = asb.BlockedSpmm(g, var, cuts)
            for k in range(bp.n_blocks):
                bp.run(k, b, c)
            torch.cuda.synchronize()
            want = oracle.spmm_baseline(m, b.cpu().numpy())
            assert bit_equal(c.cpu().numpy(), want), (name, var)
            bp.close()
        g.close()


@pytest.mark.parametrize("dt", [torch.bfloat16, torch.float16])
def test_half_ops_degenerate(dt):
    rng = np.random.default_rng(97)
    for name, m in shapes():
        if m.n_rows == 0:
            continue
        crow = torch.from_numpy(m.rowptr.astype(np.int64)).cuda()
        col = torch.from_numpy(m.colind.astype(np.int32)).cuda()
        val = torch.from_numpy(m.val if m.val is not None else np.ones(m.nnz, np.float32)).cuda()
        b = torch.from_numpy(random_dense(rng, m.n_cols, 8)).cuda().to(dt)
        out = torch.ops.autosage.spmm_csr(crow, col, val, b, "spmm:hubsplit:ft=64:rpc=1:vec=1:hubt=1")
        want = oracle.spmm_baseline(m.with_values(val.cpu().numpy()), b.float().cpu().numpy())
        assert out.shape == (m.n_rows, 8) and bit_equal(out.cpu().numpy(), want), (name, dt)
        x = torch.from_numpy(random_dense(rng, m.n_rows, 8)).cuda().to(dt)
        y = torch.from_numpy(random_dense(rng, m.n_cols, 8)).cuda().to(dt)
        s = torch.ops.autosage.sddmm_csr(crow, col, x, y, "")
        want_s = oracle.sddmm(m.with_values(None), x.float().cpu().numpy(), y.float().cpu().numpy()) \
            if m.nnz else np.zeros(0, np.float32)
        assert s.shape == (m.nnz,) and bit_equal(s.cpu().numpy(), want_s), (name, dt)
