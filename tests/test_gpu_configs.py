"""Parity at the BASELINE.json configurations.

The small-graph suites (test_gpu_kernels.py, test_gpu_scheduler.py) pin every
kernel against the oracle; this module runs the paths the bench takes at
full size -- the >= 16M-nnz dispatch branch (no ring kernel, rows of up to
21,657 entries in the lane-group kernel, thousands of hub pieces), the c4
1M-nnz hubs (489 pieces, one reduce) and c5's 8 heads -- and checks them
against the reference library itself (oracle/_ref, compiled from
/root/reference; the C port where it is absent):

* c1 (100k rows, 1.6M nnz, F=64) in full, every mapping, bit for bit;
* Reddit-shape (232,965 rows, 114.6M nnz) at F = 32/64/128/256 on a row
  sample (every 128th row plus the 32 heaviest), bit for bit;
* c4's 1M / 250k / 60k-nnz hubs plus a row sample, bit for bit, and the
  scheduler's guardrail + replay on that graph;
* c5: 8 heads x F=64 attention on sampled rows, fused == staged bit for bit
  and within the reference tolerance 1e-6 + 1e-5|want|
  (proj/tests/test_util.hpp:28) of the reference's own pipeline.
"""
import os
import subprocess
import sys

import numpy as np
import pytest

import bench
import oracle
import paper_2511_17594_b200 as asb
from tests.util import bit_equal, cuda, max_err, n_bit_diff

pytestmark = pytest.mark.gpu

SP, SD = asb.SPMM, asb.SDDMM
RP, HS = asb.ROWPARALLEL, asb.HUBSPLIT


def V(op, mapping, ft=64, rpc=1, vec=True, hubt=256):
    return asb.KernelVariant(op, mapping, ft, rpc, vec, hubt)


def vs(v):
    return asb.variant_to_string(v)


class Ref:
    """The reference library on a host CSR (oracle/_ref), else the C port."""

    def __init__(self, m):
        self.m = m
        self.lib = oracle.ref_available()
        self.g = oracle.RefGraph(m) if self.lib else None

    def spmm(self, v, b):
        if self.lib:
            if v is None:
                return oracle.ref_spmm_baseline(self.g, oracle.RefDense(b))
            return oracle.ref_spmm_dispatch(vs(v), self.g, oracle.RefDense(b))[0]
        if v is not None and v.mapping == HS:
            return oracle.spmm_hubsplit(self.m, b, v.hub_threshold)
        return oracle.spmm_baseline(self.m, b)

    def sddmm(self, v, x, y):
        if self.lib:
            if v is None:
                return oracle.ref_sddmm_baseline(self.g, oracle.RefDense(x), oracle.RefDense(y))
            return oracle.ref_sddmm_dispatch(vs(v), self.g, oracle.RefDense(x), oracle.RefDense(y))
        if v is None:
            return oracle.sddmm(self.m, x, y)
        return oracle.sddmm(self.m, x, y, v.f_tile, v.vectorized)


def row_sample(m, step, heaviest=32):
    deg = np.diff(m.rowptr.astype(np.int64))
    rows = np.union1d(np.arange(0, m.n_rows, step), np.argsort(-deg, kind="stable")[:heaviest])
    return rows.astype(np.uint64)


def sliced(m, rows):
    rp, ci, va = oracle.slice_rows(m, rows)
    return oracle.HostCsr(rows.size, m.n_cols, rp, ci, va)


def entry_index(m, rows):
    """Entry positions of `rows` in m (the SDDMM outputs of a row slice)."""
    rp = m.rowptr.astype(np.int64)
    return np.concatenate([np.arange(rp[r], rp[r + 1]) for r in rows.astype(np.int64)])


# ---- c1: the reference's own CPU-runnable case, in full -----------------------
def test_c1_full_graph_every_mapping_bit_exact():
    m, f = bench.make_graph("c1", 1)
    b, x, y = bench.dense_inputs(asb.fill_uniform, m, f, 1)
    ref = Ref(m)
    g = asb.Graph.from_csr(m)
    bd, xd, yd = cuda(b), cuda(x), cuda(y)
    want = ref.spmm(None, b)
    assert bit_equal(asb.spmm_baseline(g, bd).cpu().numpy(), want)
    for ft in (32, 64, 128):
        for rpc in (1, 4, 16):
            for vec in (False, True):
                got = asb.dispatch(V(SP, RP, ft, rpc, vec), g, bd).output.cpu().numpy()
                assert bit_equal(got, want), (ft, rpc, vec, n_bit_diff(got, want))
    for hubt in (16, 64, 256, 1024, 4096):
        want_h = ref.spmm(V(SP, HS, 64, 1, True, hubt), b)
        for ft, vec in ((64, True), (32, False), (128, True)):
            got = asb.dispatch(V(SP, HS, ft, 1, vec, hubt), g, bd).output.cpu().numpy()
            assert bit_equal(got, want_h), (hubt, ft, vec, n_bit_diff(got, want_h))
    for ft, vec in ((32, False), (64, False), (32, True), (64, True)):
        want_s = ref.sddmm(V(SD, RP, ft, 1, vec), x, y)
        for mapping in (RP, HS):
            got = asb.dispatch(V(SD, mapping, ft, 4, vec), g, xd, yd).values.cpu().numpy()
            assert bit_equal(got, want_s), (ft, vec, mapping, n_bit_diff(got, want_s))
    assert bit_equal(asb.sddmm_baseline(g, xd, yd).cpu().numpy(), ref.sddmm(None, x, y))
    # the scheduler's pick on the full graph is one of the above
    c = asb.spmm_auto(g, bd).cpu().numpy()
    assert any(bit_equal(c, ref.spmm(V(SP, HS, 64, 1, True, t), b)) for t in (256,)) or bit_equal(c, want)


# ---- c2: Reddit-shape, 114.6M nnz (the >= 16M-nnz dispatch branch) -------------
@pytest.fixture(scope="module")
def reddit():
    m, _ = bench.make_graph("reddit", 1)
    g = asb.Graph.from_csr(m)
    rows = row_sample(m, 128)
    yield m, g, rows, sliced(m, rows), entry_index(m, rows)
    g.close()


@pytest.mark.parametrize("f", [32, 64, 128, 256])
def test_reddit_shape_sampled_rows_bit_exact(reddit, f):
    m, g, rows, ms, eidx = reddit
    b, x, y = bench.dense_inputs(asb.fill_uniform, m, f, 1)
    bd, xd, yd = cuda(b), cuda(x), cuda(y)
    ref = Ref(ms)
    ridx = rows.astype(np.int64)
    want_rows = ref.spmm(None, b)
    got = asb.spmm_baseline(g, bd).cpu().numpy()[ridx]
    assert bit_equal(got, want_rows), n_bit_diff(got, want_rows)
    # row mode: every row (up to 21,657 entries) in the lane-group kernel
    for ft in sorted({min(64, f), f}):
        got = asb.dispatch(V(SP, RP, ft, 1, True), g, bd).output.cpu().numpy()[ridx]
        assert bit_equal(got, want_rows), (ft, n_bit_diff(got, want_rows))
    # hub-split as the bench decides it (thousands of 2048-entry pieces)
    for hubt in (256, 4096):
        want_h = ref.spmm(V(SP, HS, 64, 1, True, hubt), b)
        for ft in sorted({min(64, f), min(128, f)}):
            got = asb.dispatch(V(SP, HS, ft, 1, True, hubt), g, bd).output.cpu().numpy()[ridx]
            assert bit_equal(got, want_h), (hubt, ft, n_bit_diff(got, want_h))
    xs = np.ascontiguousarray(x[ridx])
    for ft, vec in ((32, False), (32, True), (64, True)):
        want_s = ref.sddmm(V(SD, RP, ft, 1, vec), xs, y)
        got = asb.dispatch(V(SD, RP, ft, 1, vec), g, xd, yd).values.cpu().numpy()[eidx]
        assert bit_equal(got, want_s), (ft, vec, n_bit_diff(got, want_s))


# ---- c4: Zipf skew with 1M / 250k / 60k-nnz hubs ---------------------------------
@pytest.fixture(scope="module")
def skew():
    m = bench.with_hubs(asb.gen_powerlaw(1_100_000, 1_100_000, 24_000_000, 2.0, 4, 1_000_000, 7),
                  [1_000_000, 250_000, 60_000], 11)
    g = asb.Graph.from_csr(m)
    rows = row_sample(m, 1024, heaviest=8)
    yield m, g, rows, sliced(m, rows)
    g.close()


@pytest.mark.parametrize("f", [16, 64, 128])
def test_c4_million_nnz_hub_bit_exact(skew, f):
    m, g, rows, ms = skew
    assert int(np.diff(m.rowptr.astype(np.int64)).max()) == 1_000_000
    b = asb.fill_uniform(m.n_cols * f, 1 + f, (m.n_cols, f))
    bd = cuda(b)
    ref = Ref(ms)
    ridx = rows.astype(np.int64)
    for hubt in (256, 4096):
        want = ref.spmm(V(SP, HS, 64, 1, True, hubt), b)
        got = asb.dispatch(V(SP, HS, min(64, f), 1, True, hubt), g, bd).output.cpu().numpy()[ridx]
        assert bit_equal(got, want), (hubt, n_bit_diff(got, want))
    assert bit_equal(asb.spmm_baseline(g, bd).cpu().numpy()[ridx], ref.spmm(None, b))


def test_c4_guardrail_and_replay_on_the_skew_graph(skew):
    m, g, _, _ = skew
    f = 64
    bd = cuda(asb.fill_uniform(m.n_cols * f, 65, (m.n_cols, f)))
    cache = asb.ScheduleCache()
    d = asb.decide_spmm(g, bd, asb.ProbeConfig(), asb.ScheduleContext(cache=cache))
    assert d.source_name == "probed"
    # guardrail (src/scheduler.cpp:156-160): a choice only if t* <= alpha * t_b
    if d.choice is not None:
        assert d.t_star <= d.alpha * d.baseline_ms
    rp = asb.decide_spmm(g, bd, asb.ProbeConfig(),
                         asb.ScheduleContext(cache=cache, replay=asb.ReplayPolicy(True, True)))
    assert rp.source_name == "replayed" and rp.choice_string() == d.choice_string()


# ---- c5: 8 heads x F=64 attention on the Reddit-shape graph ----------------------
def test_c5_eight_head_attention_sampled_rows(reddit):
    m, g, rows, ms, _ = reddit
    f = 64
    ridx = rows.astype(np.int64)
    pat = oracle.HostCsr(ms.n_rows, ms.n_cols, ms.rowptr, ms.colind, None)
    cache = asb.ScheduleCache()
    for h in range(8):
        q = asb.fill_uniform(m.n_rows * f, 1 + 3 * h, (m.n_rows, f))
        k = asb.fill_uniform(m.n_cols * f, 2 + 3 * h, (m.n_cols, f))
        v = asb.fill_uniform(m.n_cols * f, 3 + 3 * h, (m.n_cols, f))
        qd, kd, vd = cuda(q), cuda(k), cuda(v)
        ctx = asb.ScheduleContext(cache=cache)
        fused = asb.csr_attention_forward(g, qd, kd, vd, ctx=ctx, fused=True).cpu().numpy()[ridx]
        staged = asb.csr_attention_forward(g, qd, kd, vd, ctx=ctx, fused=False).cpu().numpy()[ridx]
        assert bit_equal(fused, staged), h
        qs = np.ascontiguousarray(q[ridx])
        if oracle.ref_available():
            want = oracle.ref_attention(oracle.RefGraph(pat), oracle.RefDense(qs), oracle.RefDense(k),
                                        oracle.RefDense(v))
        else:
            want = oracle.attention(pat, qs, k, v)
        assert max_err(fused, want) <= 1.0, h


# ---- the large-graph dispatch branch, forced on a small graph ---------------------
_FORCED = r'''
import numpy as np, oracle, paper_2511_17594_b200 as asb
from tests.util import hub_graph, random_dense, bit_equal, cuda
rng = np.random.default_rng(91)
# 900 rows of degree 300..1200 (900 pieces > 4 x 148: the lane-group pieces
# path) + light rows; 6000 columns
deg = np.concatenate([rng.integers(300, 1200, 900), rng.integers(0, 40, 7100)])
from tests.util import csr_from_degrees
a = csr_from_degrees(rng, 8000, 6000, deg)
for f in (32, 64, 100):
    b = random_dense(rng, 6000, f)
    g = asb.Graph.from_csr(a)
    bd = cuda(b)
    want = oracle.spmm_baseline(a, b)
    for ft, vec in ((64, True), (32, False)):
        got = asb.dispatch(asb.KernelVariant(asb.SPMM, asb.ROWPARALLEL, ft, 1, vec), g, bd).output
        assert bit_equal(got.cpu().numpy(), want), ("rows", f, ft, vec)
    for hubt in (64, 256):
        want_h = oracle.spmm_hubsplit(a, b, hubt)
        got = asb.dispatch(asb.KernelVariant(asb.SPMM, asb.HUBSPLIT, 64, 1, True, hubt), g, bd).output
        assert bit_equal(got.cpu().numpy(), want_h), ("hub", f, hubt)
    g.close()
print("FORCED_OK")
'''


@pytest.mark.parametrize("long_row", ["4611686018427387904", "0", "256"])
def test_large_graph_dispatch_branch_forced(long_row):
    """AUTOSAGE_DEV_LONG_ROW: 2^62 = no ring kernel (what a >= 16M-nnz graph
    runs), 0 = disabled, 256 = the small-graph default.  The knob is read
    once per process, so each setting runs in its own interpreter."""
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, AUTOSAGE_DEV_LONG_ROW=long_row, PYTHONPATH=root)
    r = subprocess.run([sys.executable, "-c", _FORCED], cwd=root, env=env, capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0 and "FORCED_OK" in r.stdout, r.stdout[-2000:] + r.stderr[-3000:]
