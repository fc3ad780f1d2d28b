"""GPU parity of the sm_100a operators against the CPU oracle.

Bar: SpMM (every mapping) and SDDMM (every variant order) are
bit-exact against the reference arithmetic restated in oracle/oracle.c;
row-softmax and attention are held to the reference tolerance
|got-want| <= 1e-6 + 1e-5|want| (proj/tests/test_util.hpp:28) and, in
practice, to <= 1 f32 ulp (the only source of difference is CUDA's f64 exp
vs libm's).  Mirrors proj/tests/test_kernels.cpp case by case.
"""
import numpy as np
import pytest

import oracle
import paper_2511_17594_b200 as asb
from tests.util import (bit_equal, cuda, empty_rows, hub_graph, identity, max_err, n_bit_diff,
                        random_csr, random_dense, ulp_diff)

pytestmark = pytest.mark.gpu

SP, SD = asb.SPMM, asb.SDDMM
RP, HS, BL = asb.ROWPARALLEL, asb.HUBSPLIT, asb.BASELINE


def V(op, mapping, ft=64, rpc=4, vec=False, hubt=256):
    return asb.KernelVariant(op, mapping, ft, rpc, vec, hubt)


# ---- SpMM: known answers (proj/tests/test_kernels.cpp:43-81) ----------------
def test_spmm_identity_passes_b_through():
    rng = np.random.default_rng(1)
    b = random_dense(rng, 2, 5)
    assert bit_equal(asb.spmm_baseline(identity(2), b), b)


def test_spmm_worked_2x2_example():
    a = asb.CsrMatrix(2, 2, [0, 1, 1], [1], np.array([2.0], np.float32))
    b = np.array([[1, 1], [3, 4]], np.float32)
    c = asb.spmm_baseline(a, b)
    assert c.tolist() == [[6.0, 8.0], [0.0, 0.0]]


def test_spmm_all_empty_rows_give_zeros():
    rng = np.random.default_rng(2)
    b = random_dense(rng, 4, 7)
    for v in (None, V(SP, RP, 32, 4, True), V(SP, HS, 64, 1, False, 1)):
        c = asb.spmm_baseline(empty_rows(3, 4), b) if v is None else \
            asb.dispatch(v, empty_rows(3, 4), b).output
        assert np.all(c == 0.0) and not np.any(np.signbit(c))


@pytest.mark.parametrize("f", [1, 2, 4, 33, 63, 64, 100, 128, 256, 300])
def test_spmm_every_variant_bit_exact_vs_oracle(f):
    rng = np.random.default_rng(3 + f)
    a = random_csr(rng, 200, 150, 40)
    b = random_dense(rng, 150, f)
    want = oracle.spmm_baseline(a, b)
    g = asb.Graph.from_csr(a)
    bd = cuda(b)
    assert bit_equal(asb.spmm_baseline(g, bd).cpu().numpy(), want)
    for ft in (1, 16, 32, 64, 128, 1024):
        for rpc in (1, 4, 16):
            for vec in (False, True):
                got = asb.dispatch(V(SP, RP, ft, rpc, vec), g, bd).output.cpu().numpy()
                assert bit_equal(got, want), (ft, rpc, vec, n_bit_diff(got, want))


def test_spmm_pattern_only_uses_implicit_one():
    rng = np.random.default_rng(4)
    a = random_csr(rng, 80, 60, 20, with_values=False)
    b = random_dense(rng, 60, 64)
    want = oracle.spmm_baseline(a, b)
    for v in (V(SP, RP, 64, 4, True), V(SP, HS, 32, 1, False, 8)):
        assert bit_equal(asb.dispatch(v, a, b).output, want)
    assert bit_equal(asb.spmm_baseline(a, b), want)


def test_spmm_identity_exact_for_every_tile():
    rng = np.random.default_rng(4)
    b = random_dense(rng, 40, 64)
    for ft in (32, 64, 128):
        assert bit_equal(asb.spmm_rowparallel(identity(40), b, V(SP, RP, ft, 4, False)), b)


@pytest.mark.parametrize("hub_t", [1, 8, 128, 256, 2048, 5000])
@pytest.mark.parametrize("f", [16, 63, 64, 128])
def test_spmm_hubsplit_bit_exact_vs_oracle(hub_t, f):
    rng = np.random.default_rng(5 + hub_t + f)
    a = hub_graph(rng, 6000, [5000, 4097, 2049, 2048, 600, 256], 6)
    b = random_dense(rng, 6000, f)
    want = oracle.spmm_hubsplit(a, b, hub_t)
    g = asb.Graph.from_csr(a)
    bd = cuda(b)
    for vec in (False, True):
        for ft in (32, 128):
            got = asb.dispatch(V(SP, HS, ft, 4, vec, hub_t), g, bd).output.cpu().numpy()
            assert bit_equal(got, want), (vec, ft, n_bit_diff(got, want))


@pytest.mark.parametrize("mode", ["2", "0"])
def test_spmm_hubsplit_one_launch_bit_exact(monkeypatch, mode):
    """Hub pieces and light rows as one item list in one launch (forced with
    AUTOSAGE_DEV_SPMM_MERGED=2 on graphs small enough for the ring kernel;
    0 = the two-kernel form): empty rows, one-entry rows, multi-piece hubs,
    f32 / bf16 B, vec and scalar tiles -- bit-equal to the oracle."""
    import torch
    import paper_2511_17594_b200.torch_ops  # noqa: F401  (torch.ops.autosage)
    monkeypatch.setenv("AUTOSAGE_DEV_SPMM_MERGED", mode)
    rng = np.random.default_rng(57)
    n = 3000
    deg = rng.choice([0, 0, 1, 3, 17, 40], size=n).astype(np.int64)
    deg[:5] = [2900, 2049, 2048, 700, 256]
    from tests.util import csr_from_degrees
    a = csr_from_degrees(rng, n, n, deg, True)
    g = asb.Graph.from_csr(a)
    for f in (4, 64, 100):
        b = random_dense(rng, n, f)
        bd = cuda(b)
        for hub_t in (1, 256):
            want = oracle.spmm_hubsplit(a, b, hub_t)
            for vec in (False, True):
                got = asb.dispatch(V(SP, HS, 64, 1, vec, hub_t), g, bd).output.cpu().numpy()
                assert bit_equal(got, want), (mode, f, hub_t, vec, n_bit_diff(got, want))
        if f == 64:  # bf16 B words through the same item list
            b16 = bd.to(torch.bfloat16)
            crow = torch.from_numpy(a.rowptr.astype(np.int64)).cuda()
            col = torch.from_numpy(a.colind.astype(np.int32)).cuda()
            got = torch.ops.autosage.spmm_csr(crow, col, cuda(a.val), b16, "spmm:hubsplit:ft=64:rpc=1:vec=1:hubt=256")
            assert bit_equal(got.cpu().numpy(), oracle.spmm_hubsplit(a, b16.float().cpu().numpy(), 256)), mode
    g.close()


def test_spmm_hubsplit_unreachable_threshold_equals_rowparallel():
    rng = np.random.default_rng(6)
    a = random_csr(rng, 128, 128, 10)
    b = random_dense(rng, 128, 32)
    hub = asb.spmm_hubsplit(a, b, V(SP, HS, 32, 4, False, (1 << 64) - 1))
    row = asb.spmm_rowparallel(a, b, V(SP, RP, 32, 4, False))
    assert bit_equal(hub, row)


def test_spmm_hubsplit_threshold_one_matches_dense_oracle():
    rng = np.random.default_rng(7)
    a = random_csr(rng, 100, 100, 40)
    b = random_dense(rng, 100, 33)
    dense = np.zeros((100, 100))
    for i in range(100):
        dense[i, a.row_cols(i)] = a.row_vals(i)
    got = asb.spmm_hubsplit(a, b, V(SP, HS, 64, 4, False, 1))
    assert max_err(got, dense @ b.astype(np.float64)) <= 1.0


def test_spmm_deterministic_across_runs():
    rng = np.random.default_rng(8)
    a = hub_graph(rng, 3000, [2500, 2500], 8)
    b = random_dense(rng, 3000, 64)
    g = asb.Graph.from_csr(a)
    bd = cuda(b)
    v = V(SP, HS, 64, 4, True, 128)
    c1 = asb.dispatch(v, g, bd).output.cpu().numpy()
    c2 = asb.dispatch(v, g, bd).output.cpu().numpy()
    assert bit_equal(c1, c2)


def test_spmm_nan_and_inf_propagate_like_the_reference():
    rng = np.random.default_rng(9)
    a = random_csr(rng, 50, 40, 10)
    b = random_dense(rng, 40, 8)
    b[3, 2] = np.nan
    b[7, 5] = np.inf
    want = oracle.spmm_baseline(a, b)
    for v in (V(SP, RP, 64, 4, True), V(SP, HS, 32, 1, False, 2)):
        got = asb.dispatch(v, a, b).output
        assert bit_equal(np.nan_to_num(got), np.nan_to_num(want))
        assert np.array_equal(np.isnan(got), np.isnan(want))


# ---- SDDMM (proj/tests/test_kernels.cpp:158-240) --------------------------------
def test_sddmm_identity_gives_row_norms():
    rng = np.random.default_rng(10)
    x = random_dense(rng, 6, 17)
    out = asb.sddmm_baseline(identity(6), x, x)
    want = np.sum(x.astype(np.float64) ** 2, axis=1)
    assert max_err(out, want) <= 1.0


def test_sddmm_edge_cases():
    rng = np.random.default_rng(11)
    p = random_csr(rng, 8, 9, 5, with_values=False)
    zero = np.zeros((8, 4), np.float32)
    y = random_dense(rng, 9, 4)
    assert np.all(asb.sddmm_baseline(p, zero, y) == 0.0)
    one = asb.CsrMatrix(1, 1, [0, 1], [0])
    out = asb.sddmm_baseline(one, np.array([[2.0]], np.float32), np.array([[3.0]], np.float32))
    assert out.tolist() == [6.0]


def test_sddmm_ignores_pattern_values():
    rng = np.random.default_rng(12)
    p = random_csr(rng, 20, 20, 6)
    x, y = random_dense(rng, 20, 8), random_dense(rng, 20, 8)
    assert bit_equal(asb.sddmm_baseline(p, x, y), asb.sddmm_baseline(p.with_values(None), x, y))


@pytest.mark.parametrize("f", [1, 3, 4, 17, 32, 63, 64, 100, 128, 256, 520])
def test_sddmm_every_variant_bit_exact_vs_oracle(f):
    rng = np.random.default_rng(13 + f)
    p = hub_graph(rng, 700, [650, 300, 64], 9, with_values=False)
    x, y = random_dense(rng, 700, f), random_dense(rng, 700, f)
    g = asb.Graph.from_csr(p)
    xd, yd = cuda(x), cuda(y)
    want_seq = oracle.sddmm(p, x, y, 64, False)
    assert bit_equal(asb.sddmm_baseline(g, xd, yd).cpu().numpy(), want_seq)
    for mapping in (RP, HS):
        for ft in (3, 16, 32, 64, 128):
            for rpc in (1, 4, 16):
                for vec in (False, True):
                    got = asb.dispatch(V(SD, mapping, ft, rpc, vec), g, xd, yd).values
                    got = got.cpu().numpy()
                    gate = vec and f % 4 == 0
                    want = oracle.sddmm(p, x, y, ft, True) if gate else want_seq
                    assert bit_equal(got, want), (mapping, ft, rpc, vec, n_bit_diff(got, want))


@pytest.mark.parametrize("f", [16, 32, 64, 128])
def test_sddmm_special_values_bit_exact(f):
    """Zeros, subnormals, huge magnitudes (exercise the ALU re-bias widening
    when Y is finite), then inf/NaN in X and in Y (the all-F2F path)."""
    rng = np.random.default_rng(40 + f)
    p = hub_graph(rng, 500, [480, 200], 6, with_values=False)
    x, y = random_dense(rng, 500, f), random_dense(rng, 500, f)
    y[::7, ::3] = 0.0
    y[1::5, 2::4] = np.float32(1e-41)  # subnormal
    y[2::9, 3::4] = np.float32(-3.0e38)
    x[::11, 2::4] = np.float32(2.5e38)
    x[3::13, ::5] = np.float32(-1e-40)
    g = asb.Graph.from_csr(p)
    cases = [(x, y)]
    x2 = x.copy()
    x2[4, 1] = np.inf
    cases.append((x2, y))
    y2 = y.copy()
    y2[5, 2], y2[9, 3] = np.nan, -np.inf
    cases.append((x, y2))
    for xx, yy in cases:
        for vec, ft in ((False, 64), (True, 32), (True, 64)):
            got = asb.dispatch(V(SD, RP, ft, 4, vec), g, cuda(xx), cuda(yy)).values.cpu().numpy()
            want = oracle.sddmm(p, xx, yy, ft, vec)
            assert np.array_equal(np.isnan(got), np.isnan(want))
            assert bit_equal(np.nan_to_num(got), np.nan_to_num(want)), (vec, ft)


@pytest.mark.parametrize("force", ["1", "0"])
def test_sddmm_pass_major_bit_exact(monkeypatch, force):
    """F >= 128 in one launch per 64-feature pass, each entry's f64 chain
    carried between launches (sddmm_pair1_pm_kernel; forced on small graphs,
    auto only when Y overflows the L2): sequential order and the ft 32 / 64
    four-way blocks, special values, chunks spanning many rows -- bit-equal
    to the oracle and to the single-launch kernel."""
    monkeypatch.setenv("AUTOSAGE_DEV_SDDMM_PM", force)
    rng = np.random.default_rng(47)
    n = 1500
    deg = rng.choice([0, 1, 2, 9], size=n).astype(np.int64)
    deg[:3] = [1400, 700, 65]
    rp = np.zeros(n + 1, np.uint64)
    rp[1:] = np.cumsum(deg)
    cols = np.concatenate([np.sort(rng.choice(n, size=d, replace=False)) for d in deg]).astype(np.uint32)
    p = asb.CsrMatrix(n, n, rp, cols, None)
    g = asb.Graph.from_csr(p)
    for f in (128, 192, 256):
        x, y = random_dense(rng, n, f), random_dense(rng, n, f)
        y[1::5, 2::4] = np.float32(1e-41)
        x[::11, 2::4] = np.float32(2.5e38)
        y2 = y.copy()
        y2[5, 70] = np.nan
        for yy in (y, y2):
            for vec, ft in ((False, 64), (True, 32), (True, 64)):
                got = asb.dispatch(V(SD, RP, ft, 4, vec), g, cuda(x), cuda(yy)).values.cpu().numpy()
                want = oracle.sddmm(p, x, yy, ft, vec)
                assert np.array_equal(np.isnan(got), np.isnan(want))
                assert bit_equal(np.nan_to_num(got), np.nan_to_num(want)), (f, vec, ft)


def test_small_work_scan_rule_keeps_bits(monkeypatch):
    """The default skips the finite scan (and the ALU re-bias widening) for
    ops under 2^28 entry-features; forcing the scan gives the same bits for
    SpMM (every mapping) and SDDMM (both orders)."""
    rng = np.random.default_rng(51)
    a = hub_graph(rng, 3000, [2900, 1200, 300], 12)
    g = asb.Graph.from_csr(a)
    b, x = random_dense(rng, 3000, 64), random_dense(rng, 3000, 64)
    outs = []
    for knob in ("0", None):
        if knob is None:
            monkeypatch.delenv("AUTOSAGE_DEV_MIX_MIN_WORK")
        else:
            monkeypatch.setenv("AUTOSAGE_DEV_MIX_MIN_WORK", knob)
        r = [asb.dispatch(V(SP, m, ft, 4, True, 256), g, cuda(b)).output.cpu().numpy()
             for m, ft in ((RP, 64), (HS, 64), (HS, 32))]
        r += [asb.dispatch(V(SD, RP, 32, 1, vec), g, cuda(x), cuda(b)).values.cpu().numpy() for vec in (False, True)]
        outs.append(r)
    for u, v in zip(*outs):
        assert bit_equal(u, v)
    assert bit_equal(outs[1][0], oracle.spmm_baseline(a, b))
    g.close()


def test_sddmm_chunks_spanning_many_rows():
    """Degree-0/1/2 rows: one 32-entry chunk meets more than 32 rows."""
    rng = np.random.default_rng(44)
    n = 3000
    deg = rng.choice([0, 1, 1, 2], size=n).astype(np.int64)
    deg[1500] = 700
    rp = np.zeros(n + 1, np.uint64)
    rp[1:] = np.cumsum(deg)
    cols = np.concatenate([np.sort(rng.choice(n, size=d, replace=False)) for d in deg]).astype(np.uint32)
    p = asb.CsrMatrix(n, n, rp, cols, None)
    g = asb.Graph.from_csr(p)
    for f in (32, 64):
        x, y = random_dense(rng, n, f), random_dense(rng, n, f)
        for vec in (False, True):
            got = asb.dispatch(V(SD, RP, 64, 4, vec), g, cuda(x), cuda(y)).values.cpu().numpy()
            assert bit_equal(got, oracle.sddmm(p, x, y, 64, vec)), (f, vec)


def test_sddmm_vec_and_scalar_stay_close():
    rng = np.random.default_rng(13)
    p = random_csr(rng, 70, 50, 9, with_values=False)
    x, y = random_dense(rng, 70, 64), random_dense(rng, 50, 64)
    ref = asb.sddmm_baseline(p, x, y)
    s = asb.sddmm_rowparallel(p, x, y, V(SD, RP, 32, 4, False))
    v = asb.sddmm_rowparallel(p, x, y, V(SD, RP, 32, 4, True))
    assert max_err(s, ref) <= 1.0 and max_err(v, ref) <= 1.0
    assert max_err(v, s, 1e-6, 1e-7) <= 1.0
    empty = empty_rows(4, 50)
    assert asb.sddmm_rowparallel(empty, np.zeros((4, 64), np.float32), y,
                                 V(SD, RP, 32, 4, False)).size == 0


def test_sddmm_duality_full_row_matches_gram():
    rng = np.random.default_rng(14)
    m = 37
    p = asb.CsrMatrix(1, m, [0, m], np.arange(m))
    x, y = random_dense(rng, 1, 24), random_dense(rng, m, 24)
    out = asb.sddmm_baseline(p, x, y)
    assert max_err(out, (x.astype(np.float64) @ y.astype(np.float64).T).ravel()) <= 1.0


# ---- row softmax (proj/tests/test_kernels.cpp:242-297) --------------------------
def test_row_softmax_basics():
    m = asb.CsrMatrix(3, 4, [0, 1, 3, 5], [0, 0, 1, 2, 3],
                      np.array([1000.0, 2.5, 2.5, 1000.0, 1001.0], np.float32))
    sm = asb.row_softmax(m)
    assert sm.val[0] == pytest.approx(1.0)
    assert sm.val[1] == pytest.approx(0.5) and sm.val[2] == pytest.approx(0.5)
    assert sm.val[3] == pytest.approx(0.26894, rel=1e-4)
    assert sm.val[4] == pytest.approx(0.73106, rel=1e-4)
    assert np.array_equal(sm.rowptr, m.rowptr) and np.array_equal(sm.colind, m.colind)


def test_row_softmax_sums_to_one_and_shift_invariant():
    rng = np.random.default_rng(15)
    m = random_csr(rng, 300, 300, 30, with_values=False)
    vals = (rng.integers(-64000, 64001, size=m.nnz) / 64.0).astype(np.float32)
    s0 = asb.row_softmax(m.with_values(vals))
    s1 = asb.row_softmax(m.with_values(vals + np.float32(1000.0)))
    for i in range(m.n_rows):
        if m.degree(i):
            assert abs(np.sum(s0.row_vals(i).astype(np.float64)) - 1.0) <= 1e-6
    assert np.max(np.abs(s0.val.astype(np.float64) - s1.val)) <= 1e-6


def test_row_softmax_nan_and_values_required():
    m = asb.CsrMatrix(1, 2, [0, 2], [0, 1], np.array([np.nan, 1.0], np.float32))
    assert np.all(np.isnan(asb.row_softmax(m).val))
    m2 = asb.CsrMatrix(1, 2, [0, 2], [0, 1], np.array([1.0, np.nan], np.float32))
    assert np.all(np.isnan(asb.row_softmax(m2).val))
    with pytest.raises(asb.InvalidArgument):
        asb.row_softmax(m.with_values(None))


@pytest.mark.parametrize("hub", [0, 5000])
def test_row_softmax_vs_oracle(hub):
    rng = np.random.default_rng(16 + hub)
    m = hub_graph(rng, 8000, [hub] if hub else [], 40)
    vals = rng.normal(0, 8, size=m.nnz).astype(np.float32)
    got = asb.row_softmax(m.with_values(vals)).val
    want = oracle.row_softmax(m, vals)
    assert max_err(got, want) <= 1.0
    assert ulp_diff(got, want) <= 1


def _softmax_stress_graph(rng):
    """Warp-path rows (<= 1024 entries) and CTA-path rows (> 1024) whose
    values make the parallel-sum certificate hold (narrow range), fail
    (tiny ex next to 1.0: very wide range, subnormal ex) or see NaN/Inf."""
    m = hub_graph(rng, 6000, [5000, 3000, 1500, 1025, 1024, 600], 40, with_values=False)
    vals = rng.uniform(-1, 1, size=m.nnz).astype(np.float32)
    rp = m.rowptr.astype(np.int64)
    wide = [1, 3, 5, 10, 11]  # rows whose sums need the sequential chain
    for r in wide:
        vals[rp[r]:rp[r + 1]] = rng.uniform(-110, 0, size=rp[r + 1] - rp[r]).astype(np.float32)
    vals[rp[12]] = np.nan                 # short row with a NaN
    vals[rp[2] + 7] = np.nan              # long row with a NaN
    vals[rp[13]:rp[14]] = np.float32(-np.inf)
    vals[rp[13]] = np.float32(3.0)        # -inf entries give ex = 0
    return m, vals, wide


def test_row_softmax_parallel_sum_equals_sequential_chain(monkeypatch):
    """The certificate path (parallel f64 sum) and the reference's sequential
    chain (AUTOSAGE_DEV_SOFTMAX_SEQ=1) give the same bits on every row, on
    both the warp (<= 1024) and the CTA (> 1024 entries) kernels."""
    rng = np.random.default_rng(61)
    m, vals, _ = _softmax_stress_graph(rng)
    fast = asb.row_softmax(m.with_values(vals)).val
    monkeypatch.setenv("AUTOSAGE_DEV_SOFTMAX_SEQ", "1")
    seq = asb.row_softmax(m.with_values(vals)).val
    assert bit_equal(fast, seq)


def test_row_softmax_predeferral_keeps_bits(monkeypatch):
    """CTA-kernel rows whose value span makes the certificate fail go to the
    chain kernel before the parallel attempt (AUTOSAGE_DEV_SOFTMAX_PREDEFER
    0 / 1 / 2): spans around the -22 bound and the estimate, NaN/Inf rows --
    the same bits every way, and the oracle's values."""
    rng = np.random.default_rng(63)
    m, vals, _ = _softmax_stress_graph(rng)
    rp = m.rowptr.astype(np.int64)
    for r, lo in ((0, -21.9), (4, -22.1), (6, -16.0), (7, -90.0), (8, -30.0)):
        vals[rp[r]:rp[r + 1]] = rng.uniform(lo, 0, size=rp[r + 1] - rp[r]).astype(np.float32)
    outs = []
    for knob in ("0", "1", "2"):
        monkeypatch.setenv("AUTOSAGE_DEV_SOFTMAX_PREDEFER", knob)
        outs.append(asb.row_softmax(m.with_values(vals)).val)
    assert bit_equal(outs[0], outs[1]) and bit_equal(outs[0], outs[2])
    want = oracle.row_softmax(m, vals)
    nan = np.isnan(want)
    assert np.array_equal(np.isnan(outs[2]), nan)
    assert ulp_diff(outs[2][~nan], want[~nan]) <= 1


def test_row_softmax_written_out_exp_equals_cuda_exp(monkeypatch):
    """sm_exp (softmax.cuh) is CUDA's f64 exp instruction sequence written
    out; AUTOSAGE_DEV_SOFTMAX_LIBEXP=1 runs exp() itself.  Same bits over
    arguments from 0 down past the f32 underflow and the fast-path edge
    (-120), including exact ties, zeros, subnormal results and NaN."""
    rng = np.random.default_rng(64)
    m = hub_graph(rng, 3000, [2500, 1100], 200, with_values=False)
    vals = rng.uniform(-130, 0, size=m.nnz).astype(np.float32)
    vals[::97] = rng.uniform(-1e-3, 0, size=vals[::97].size).astype(np.float32)
    edge = np.array([-120.0, -119.99999, -103.97208, -103.27893, -87.33655, -0.0, 0.0, -1e-30,
                     -np.inf, np.nan, -126.5], np.float32)
    vals[1:1 + edge.size] = edge            # inside the long row: max(row) stays 0-ish
    rp = m.rowptr.astype(np.int64)
    for r in range(2, 3000):                # every row's max is 0, so d = v exactly
        vals[rp[r]] = 0.0
    vals[rp[0]] = 0.0
    vals[rp[1]] = 0.0
    fast = asb.row_softmax(m.with_values(vals)).val
    monkeypatch.setenv("AUTOSAGE_DEV_SOFTMAX_LIBEXP", "1")
    lib = asb.row_softmax(m.with_values(vals)).val
    assert bit_equal(np.nan_to_num(fast), np.nan_to_num(lib))
    assert np.array_equal(np.isnan(fast), np.isnan(lib))
    # the division fast path (q = ex * RN(1/sum), midpoint check) vs the
    # oracle's correctly rounded division
    want = oracle.row_softmax(m, vals)
    ok = ~np.isnan(want)
    assert ulp_diff(fast[ok], want[ok]) <= 1


def test_row_softmax_long_and_wide_rows_vs_oracle():
    rng = np.random.default_rng(62)
    m, vals, wide = _softmax_stress_graph(rng)
    got = asb.row_softmax(m.with_values(vals)).val
    want = oracle.row_softmax(m, vals)
    nan = np.isnan(want)
    assert np.array_equal(np.isnan(got), nan)
    rp = m.rowptr.astype(np.int64)
    assert np.all(nan[rp[12]:rp[13]]) and np.all(nan[rp[2]:rp[3]])
    assert max_err(got[~nan], want[~nan]) <= 1.0
    assert ulp_diff(got[~nan], want[~nan]) <= 1
    assert np.all(got[rp[13] + 1:rp[14]] == 0.0) and got[rp[13]] == 1.0


# ---- dispatch (proj/tests/test_kernels.cpp:299-363) ------------------------------
def test_dispatch_vec4_gate_and_path_marker():
    rng = np.random.default_rng(16)
    a = random_csr(rng, 32, 32, 6)
    g = asb.Graph.from_csr(a)
    v = V(SP, RP, 32, 4, True)
    aligned = cuda(random_dense(rng, 32, 64))
    assert asb.dispatch(v, g, aligned).vectorized_path
    odd = random_dense(rng, 32, 63)
    r = asb.dispatch(v, g, cuda(odd))
    assert not r.vectorized_path
    assert bit_equal(r.output.cpu().numpy(), oracle.spmm_baseline(a, odd))
    import torch
    buf = torch.zeros(32 * 64 + 2, dtype=torch.float32, device="cuda")
    under = buf[2:].view(32, 64)  # 8-byte aligned base
    under.copy_(aligned)
    assert under.data_ptr() % 16 != 0
    r2 = asb.dispatch(v, g, under)
    assert not r2.vectorized_path
    assert bit_equal(r2.output.cpu().numpy(), asb.dispatch(v, g, aligned).output.cpu().numpy())
    assert not asb.dispatch(V(SP, RP, 32, 4, False), g, aligned).vectorized_path
    assert not asb.dispatch(V(SP, BL, 32, 4, True), g, aligned).vectorized_path


def test_dispatch_rejects_op_operand_mismatch():
    rng = np.random.default_rng(17)
    a = random_csr(rng, 8, 8, 3)
    b = random_dense(rng, 8, 4)
    with pytest.raises(asb.InvalidArgument):
        asb.dispatch(V(SD, RP, 32, 4, False), a, b)
    with pytest.raises(asb.InvalidArgument):
        asb.dispatch(V(SP, RP, 32, 4, False), a, b, b)
    with pytest.raises(asb.InvalidArgument):
        asb.spmm_baseline(a, np.zeros((9, 4), np.float32))
    with pytest.raises(asb.InvalidArgument):
        asb.spmm_rowparallel(a, b, V(SP, HS, 32, 4, False))
    with pytest.raises(asb.InvalidArgument):
        asb.dispatch(V(SP, RP, 0, 4, False), a, b)


def test_dispatch_honors_kernel_env_overrides(monkeypatch):
    rng = np.random.default_rng(18)
    a = random_csr(rng, 16, 16, 4)
    b = random_dense(rng, 16, 8)
    v = V(SP, RP, 64, 4, False)
    monkeypatch.setenv("AUTOSAGE_FTILE", "16")
    monkeypatch.setenv("AUTOSAGE_WPB", "2")
    r = asb.dispatch(v, a, b)
    monkeypatch.delenv("AUTOSAGE_FTILE")
    monkeypatch.delenv("AUTOSAGE_WPB")
    assert r.variant.f_tile == 16 and r.variant.rows_per_chunk == 2
    plain = asb.dispatch(v, a, b)
    assert plain.variant.f_tile == 64
    assert bit_equal(r.output, plain.output)


def test_dispatch_reports_elapsed_time():
    rng = np.random.default_rng(19)
    a = random_csr(rng, 500, 500, 50)
    r = asb.dispatch(V(SP, RP, 64, 4, True), asb.Graph.from_csr(a), cuda(random_dense(rng, 500, 64)))
    assert r.elapsed_ms > 0.0


# ---- attention kernels (fused / unfused) -------------------------------------------
@pytest.mark.parametrize("fused", [False, True])
@pytest.mark.parametrize("f,fv", [(16, 16), (64, 64), (64, 100), (128, 32)])
def test_attention_vs_oracle(fused, f, fv):
    rng = np.random.default_rng(20 + f + fv)
    p = hub_graph(rng, 3000, [2600, 900], 12, with_values=False)
    q, k, v = random_dense(rng, 3000, f), random_dense(rng, 3000, f), random_dense(rng, 3000, fv)
    ctx = asb.ScheduleContext(device=asb.DeviceProfile.fixed(20e9, 40e9, 2, "test"),
                              cache=asb.ScheduleCache())
    run = asb.attention_probe_breakdown(p, q, k, v, asb.ProbeConfig(iters=2), ctx, fused=fused)
    sd, pd = run.sddmm_decision, run.spmm_decision
    sv = sd.choice
    s_vec = sv is not None and sv.vectorized and f % 4 == 0
    hub_t = pd.choice.hub_threshold if (pd.choice and pd.choice.mapping == HS) else 0
    want = oracle.attention(p, q, k, v, sv.f_tile if sv else 64, s_vec, hub_t)
    assert max_err(run.output, want) <= 1.0
    assert ulp_diff(run.output, want) <= 2


def test_fused_attention_equals_unfused_bitwise():
    rng = np.random.default_rng(21)
    p = hub_graph(rng, 5000, [4500, 2100, 700], 30, with_values=False)
    q, k, v = (random_dense(rng, 5000, 64) for _ in range(3))
    cache = asb.ScheduleCache()
    ctx = asb.ScheduleContext(device=asb.DeviceProfile.fixed(20e9, 40e9, 2, "test"), cache=cache)
    cold = asb.attention_probe_breakdown(p, q, k, v, asb.ProbeConfig(iters=2), ctx)
    warm = asb.attention_probe_breakdown(p, q, k, v, asb.ProbeConfig(iters=2), ctx, fused=True)
    assert warm.sddmm_decision.source == asb.CACHED
    assert bit_equal(cold.output, warm.output)


@pytest.mark.parametrize("force", [("AUTOSAGE_WPB", "4"), ("AUTOSAGE_HUB_T", "256"),
                                   ("AUTOSAGE_HUB_T", "1"), ("AUTOSAGE_FTILE", "32"),
                                   ("AUTOSAGE_DEV_SPMM_MERGED", "2")])
@pytest.mark.parametrize("scale", [1.0, 40.0])
def test_fused_attention_softmax_on_the_fly_bitwise(monkeypatch, force, scale):
    """Fused path = SDDMM -> per-row (max, sum) -> SpMM computing each
    probability as it loads the score.  Same bits as the staged pipeline for
    row-parallel and hub-split SpMM (pieces, long rows, light rows), and for
    score ranges wide enough that row sums take the sequential chain."""
    monkeypatch.setenv(*force)  # a mapped SpMM variant (the fused path needs one)
    rng = np.random.default_rng(63)
    p = hub_graph(rng, 4000, [3900, 2049, 1500, 300], 25, with_values=False)
    q = random_dense(rng, 4000, 64) * np.float32(scale)
    k, v = random_dense(rng, 4000, 64), random_dense(rng, 4000, 32)
    cache = asb.ScheduleCache()
    ctx = asb.ScheduleContext(device=asb.DeviceProfile.fixed(20e9, 40e9, 2, "test"), cache=cache)
    staged = asb.attention_probe_breakdown(p, q, k, v, asb.ProbeConfig(iters=2), ctx, fused=False)
    fused = asb.attention_probe_breakdown(p, q, k, v, asb.ProbeConfig(iters=2), ctx, fused=True)
    assert fused.spmm_decision.choice is not None
    assert bit_equal(staged.output, fused.output)


# ---- host-buffer pipeline (as_*_host, as_*_host_async) ------------------------------
@pytest.mark.parametrize("slices,head", [("1", "8"), ("3", "1"), ("3", "8"), ("8", "8"), ("8", "1000"),
                                         ("1000000", "8")])
def test_sddmm_host_slices_bit_exact(monkeypatch, slices, head):
    """The SDDMM values leave in slices of 32-entry chunks (the first one
    1/head of the rest); every slicing returns the same bytes (odd nnz,
    fixed-width and generic widths)."""
    monkeypatch.setenv("AUTOSAGE_HOST_SLICES", slices)
    monkeypatch.setenv("AUTOSAGE_HOST_HEAD", head)
    monkeypatch.setenv("AUTOSAGE_DEV_SDDMM_PM", "1")  # F=128: pass-major per slice
    rng = np.random.default_rng(51)
    p = hub_graph(rng, 900, [850, 333, 70], 7, with_values=False)
    assert p.nnz % 32 != 0
    g = asb.Graph.from_csr(p)
    for f in (64, 24, 128):
        x, y = random_dense(rng, 900, f), random_dense(rng, 900, f)
        for v in (None, V(SD, RP, 64, 4, True), V(SD, HS, 32, 1, False)):
            got = asb.sddmm_baseline(g, x, y) if v is None else asb.dispatch(v, g, x, y).values
            want = oracle.sddmm(p, x, y, 64 if v is None else v.f_tile, v is not None and v.vectorized)
            assert bit_equal(got, want), (f, v)


def test_host_async_spmm_and_sddmm_in_flight_together():
    """Several async SpMM + SDDMM calls queued on one graph before a single
    synchronize: per-op staging and event ordering keep every result exact."""
    import torch
    rng = np.random.default_rng(52)
    a = hub_graph(rng, 1200, [1100, 700, 90], 8)
    g = asb.Graph.from_csr(a)
    f = 32
    pin = lambda arr: torch.from_numpy(arr).pin_memory().numpy()  # noqa: E731
    bs = [pin(random_dense(rng, 1200, f)) for _ in range(3)]
    xs = [pin(random_dense(rng, 1200, f)) for _ in range(3)]
    ys = [pin(random_dense(rng, 1200, f)) for _ in range(3)]
    cs = [pin(np.zeros((1200, f), np.float32)) for _ in range(3)]
    outs = [pin(np.zeros(a.nnz, np.float32)) for _ in range(3)]
    vs = V(SP, HS, 32, 4, True, 256)
    vd = V(SD, RP, 32, 4, True)
    for i in range(3):
        asb.spmm_host_async(vs, g, bs[i], cs[i])
        asb.sddmm_host_async(vd, g, xs[i], ys[i], outs[i])
    g.synchronize()
    for i in range(3):
        assert bit_equal(cs[i], oracle.spmm_hubsplit(a, bs[i], 256))
        assert bit_equal(outs[i], oracle.sddmm(a, xs[i], ys[i], 32, True))
