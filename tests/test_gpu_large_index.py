"""Maximum-size addressing: a dense operand past 2^32 elements (70M rows x
F=64 = 17.9 GB), so the gather offsets col*F no longer fit 32 bits -- the
SpMM lane-group kernels leave their one-IMAD 32-bit fast path
(fast_gather_ok) and every SDDMM kernel must form 64-bit row addresses.
Entries hit columns on both sides of the 2^32/F boundary; results must
equal the oracle bit for bit (computed on the referenced rows only)."""
import numpy as np
import pytest
import torch

import oracle
import paper_2511_17594_b200 as asb
from tests.util import bit_equal

pytestmark = pytest.mark.gpu

N_COLS = 70_000_000
F = 64


def V(op, mapping, ft=64, rpc=1, vec=True, hubt=256):
    return asb.KernelVariant(op, mapping, ft, rpc, vec, hubt)


@pytest.fixture(scope="module")
def big():
    rng = np.random.default_rng(123)
    n_rows = 600
    deg = rng.integers(0, 40, n_rows)
    deg[:2] = [3000, 700]  # hub pieces at hubT 256
    boundary = (1 << 32) // F  # first column whose col*F overflows 32 bits
    cols = []
    for d in deg:
        lo = rng.choice(np.arange(boundary - 2000, boundary + 2000), size=min(d // 2, 4000), replace=False)
        hi = rng.choice(N_COLS, size=d - lo.size, replace=False)
        cols.append(np.unique(np.concatenate([lo, hi]))[:d])
    deg = np.array([c.size for c in cols])
    rp = np.zeros(n_rows + 1, np.uint64)
    rp[1:] = np.cumsum(deg)
    ci = np.concatenate(cols).astype(np.uint32)
    val = rng.uniform(-1, 1, ci.size).astype(np.float32)
    m = asb.CsrMatrix(n_rows, N_COLS, rp, ci, val)
    # the dense operand: only the referenced rows hold data (the oracle sees
    # them compacted, same values in the same entry order)
    used, inv = np.unique(ci, return_inverse=True)
    rows_b = rng.uniform(-1, 1, (used.size, F)).astype(np.float32)
    b = torch.zeros((N_COLS, F), dtype=torch.float32, device="cuda")
    b[torch.from_numpy(used.astype(np.int64)).cuda()] = torch.from_numpy(rows_b).cuda()
    small = asb.CsrMatrix(n_rows, used.size, rp, inv.astype(np.uint32), val)
    yield m, small, b, rows_b
    del b
    torch.cuda.empty_cache()


def test_spmm_past_32bit_offsets(big):
    m, small, b, rows_b = big
    g = asb.Graph.from_csr(m)
    want = oracle.spmm_baseline(small, rows_b)
    got = asb.spmm_baseline(g, b).cpu().numpy()
    assert bit_equal(got, want)
    for v in (V(asb.SPMM, asb.ROWPARALLEL, 64, 1, True), V(asb.SPMM, asb.ROWPARALLEL, 32, 1, False)):
        assert bit_equal(asb.dispatch(v, g, b).output.cpu().numpy(), want), v
    got = asb.dispatch(V(asb.SPMM, asb.HUBSPLIT, 64, 1, True, 256), g, b).output.cpu().numpy()
    assert bit_equal(got, oracle.spmm_hubsplit(small, rows_b, 256))
    g.close()


def test_sddmm_past_32bit_offsets(big):
    m, small, y, rows_y = big
    rng = np.random.default_rng(124)
    p, ps = m.with_values(None), small.with_values(None)
    g = asb.Graph.from_csr(p)
    x = rng.uniform(-1, 1, (m.n_rows, F)).astype(np.float32)
    xd = torch.from_numpy(x).cuda()
    assert bit_equal(asb.sddmm_baseline(g, xd, y).cpu().numpy(), oracle.sddmm(ps, x, rows_y))
    for ft, vec in ((32, False), (32, True), (64, True)):
        got = asb.dispatch(V(asb.SDDMM, asb.ROWPARALLEL, ft, 1, vec), g, xd, y).values.cpu().numpy()
        assert bit_equal(got, oracle.sddmm(ps, x, rows_y, ft, vec)), (ft, vec)
    g.close()
