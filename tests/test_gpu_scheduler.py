"""Device scheduler, graph utilities and attention pipeline on the GPU.

Mirrors proj/tests/test_scheduler.cpp, test_attention.cpp, test_csr.cpp and
test_generate.cpp; features / sample / slice / graph_sig are bit-exact
against the oracle (and the reference library itself when built).
"""
import dataclasses

import numpy as np
import pytest

import oracle
import paper_2511_17594_b200 as asb
from tests.util import (FakeTimer, bit_equal, close, cuda, hub_graph, identity, max_err,
                        random_csr, random_dense)

pytestmark = pytest.mark.gpu


def fixed_dev():
    return asb.DeviceProfile.fixed(20e9, 40e9, 2, "test")


class Fixture:
    """gen_er(64, 0.1, 99)-sized graph and a 64x32 B (test_scheduler.cpp:15-42)."""

    def __init__(self):
        rng = np.random.default_rng(99)
        self.a = random_csr(rng, 64, 64, 12)
        self.b = random_dense(np.random.default_rng(100), 64, 32)
        self.dev = fixed_dev()

    def cfg(self, alpha=0.95):
        return asb.ProbeConfig(iters=1, cap_ms=1e9, top_k=3, alpha=alpha)

    def decide_with(self, timer, alpha=0.95, cache=None):
        ctx = asb.ScheduleContext(device=self.dev, timer=timer, cache=cache)
        return asb.decide_spmm(self.a, self.b, self.cfg(alpha), ctx)


# ---- graph utilities vs oracle ----------------------------------------------------
@pytest.mark.parametrize("shape", ["er", "hub", "skew", "empty_rows"])
def test_features_sample_slice_sig_bit_exact(shape):
    rng = np.random.default_rng(1)
    if shape == "er":
        m = random_csr(rng, 5000, 5000, 12)
    elif shape == "hub":
        m = hub_graph(rng, 20000, [5000], 64)
    elif shape == "skew":
        m = asb.gen_powerlaw(30000, 30000, 0, 2.1, 2, 3000, 5)
    else:
        m = random_csr(rng, 3000, 100, 3)
    g = asb.Graph.from_csr(m)
    for hub_t in (1, 32, 256):
        got = g.features(hub_t)
        want = oracle.extract_features(m, hub_t)
        for k, v in want.items():
            assert getattr(got, k) == v, k
    for frac, min_rows in ((0.02, 512), (0.05, 16), (1.0, 1), (0.5, 10**9)):
        rows = g.sample_row_indices(frac, min_rows)
        assert np.array_equal(rows, oracle.sample_row_indices(m, frac, min_rows))
        s = g.slice_rows(rows).download()
        rp, ci, va = oracle.slice_rows(m, rows)
        assert np.array_equal(s.rowptr, rp) and np.array_equal(s.colind, ci)
        assert bit_equal(s.val, va)
    assert g.sig() == oracle.graph_sig(m) == asb.graph_sig(m)


@pytest.mark.skipif(not oracle.ref_available(), reason="reference library not built")
def test_graph_utilities_match_the_reference_library():
    n_rows, n_cols, rp, ci, va = oracle.ref_gen("hub_fixed", 20000, hubs=1, hub_deg=5000,
                                                other_deg=64, seed=21)
    m = asb.CsrMatrix(n_rows, n_cols, rp, ci, va)
    rg = oracle.RefGraph(m)
    g = asb.Graph.from_csr(m)
    assert g.sig() == oracle.ref_graph_sig(rg)
    rows = g.sample_row_indices(0.02, 512)
    assert rows.size == 512 and m.degree(int(rows[0])) == 5000
    assert np.array_equal(rows, oracle.ref_sample_row_indices(rg, 0.02, 512))
    want = oracle.ref_extract_features(rg)
    got = g.features()
    for k, v in want.items():
        assert getattr(got, k) == v, k


def test_generate_sample_sizes_kat():
    # proj/tests/test_generate.cpp:91-124 sizes (2000 / 400 / 512, hub first)
    big = hub_graph(np.random.default_rng(9), 100000, [100], 4)
    assert asb.sample_row_indices(big, 0.02, 512).size == 2000
    small = hub_graph(np.random.default_rng(9), 400, [100], 4)
    assert asb.sample_row_indices(small, 0.02, 512).size == 400


# ---- scheduler with scripted timers (proj/tests/test_scheduler.cpp:70-217) ------
def test_guardrail_boundary():
    fx = Fixture()
    d = fx.decide_with(FakeTimer([10.0, 9.4, 11.0, 12.0]))
    assert d.choice is not None and d.t_star == 9.4
    assert d.source == asb.PROBED
    d = fx.decide_with(FakeTimer([10.0, 9.6, 11.0, 12.0]))
    assert d.choice is None and d.choice_string() == "baseline"
    tb = 10.0
    tie = 0.95 * tb
    d = fx.decide_with(FakeTimer([tb, tie, tie + 1.0, tie + 2.0]))
    assert d.choice is not None


def test_t_star_first_come_on_ties():
    fx = Fixture()
    d = fx.decide_with(FakeTimer([10.0, 8.0, 7.5, 7.5]))
    assert len(d.candidates) == 3
    assert d.t_star == 7.5 and d.best_index == 1
    assert d.choice == d.candidates[1].variant


def test_decide_is_pure_function_of_script():
    fx = Fixture()
    d1 = fx.decide_with(FakeTimer([10.0, 9.0, 9.3, 8.8]))
    d2 = fx.decide_with(FakeTimer([10.0, 9.0, 9.3, 8.8]))
    assert d1.choice_string() == d2.choice_string()
    assert d1.t_star == d2.t_star and d1.baseline_ms == d2.baseline_ms and d1.key == d2.key


def test_cache_hits_skip_probing():
    fx = Fixture()
    cache = asb.ScheduleCache()
    cold = fx.decide_with(FakeTimer([10.0, 9.0, 9.5, 9.8]), cache=cache)
    assert cold.source == asb.PROBED and cache.size() == 1
    asb.reset_probe_launch_count()
    warm = fx.decide_with(FakeTimer([]), cache=cache)
    assert warm.source == asb.CACHED
    assert warm.choice_string() == cold.choice_string()
    assert asb.probe_launch_count() == 0


def test_replay_mode_never_probes():
    fx = Fixture()
    cache = asb.ScheduleCache()
    ctx = asb.ScheduleContext(device=fx.dev, cache=cache,
                              replay=asb.ReplayPolicy(replay_only=True))
    asb.reset_probe_launch_count()
    d = asb.decide_spmm(fx.a, fx.b, fx.cfg(), ctx)
    assert d.source == asb.REPLAYED and d.choice is None and asb.probe_launch_count() == 0
    ctx.replay.strict = True
    with pytest.raises(asb.ReplayMiss):
        asb.decide_spmm(fx.a, fx.b, fx.cfg(), ctx)
    cold = asb.decide_spmm(fx.a, fx.b, fx.cfg(), asb.ScheduleContext(
        device=fx.dev, cache=cache, timer=FakeTimer([10.0, 9.0, 9.5, 9.8])))
    asb.reset_probe_launch_count()
    rep = asb.decide_spmm(fx.a, fx.b, fx.cfg(), ctx)
    assert rep.source == asb.REPLAYED and rep.choice_string() == cold.choice_string()
    assert asb.probe_launch_count() == 0


def test_forced_env_knobs_bypass_probe(monkeypatch):
    fx = Fixture()
    monkeypatch.setenv("AUTOSAGE_FTILE", "32")
    asb.reset_probe_launch_count()
    d = asb.decide_spmm(fx.a, fx.b, fx.cfg(), asb.ScheduleContext(device=fx.dev))
    monkeypatch.delenv("AUTOSAGE_FTILE")
    assert d.source == asb.FORCED_ENV and d.choice.f_tile == 32
    assert d.choice.mapping == asb.ROWPARALLEL and asb.probe_launch_count() == 0
    monkeypatch.setenv("AUTOSAGE_HUB_T", "128")
    h = asb.decide_spmm(fx.a, fx.b, fx.cfg(), asb.ScheduleContext(device=fx.dev))
    assert h.choice.mapping == asb.HUBSPLIT and h.choice.hub_threshold == 128


def test_probe_runs_kernels_and_counts_launches():
    fx = Fixture()
    asb.reset_probe_launch_count()
    t = FakeTimer([1.0, 0.5, 0.6, 0.7], run_kernels=True)
    d = fx.decide_with(t)
    # 4 kernels x (1 warm-up + 1 timed)
    assert asb.probe_launch_count() == 8 and t.calls() == 4
    assert d.sample_rows == 64


def test_spmm_auto_matches_baseline_kernel():
    rng = np.random.default_rng(55)
    a = hub_graph(rng, 800, [300], 6)
    b = random_dense(np.random.default_rng(101), 800, 64)
    got, d = asb.spmm_auto(a, b, asb.ProbeConfig(iters=2),
                           asb.ScheduleContext(device=fixed_dev()), return_decision=True)
    want = oracle.spmm_hubsplit(a, b, d.choice.hub_threshold) if (
        d.choice and d.choice.mapping == asb.HUBSPLIT) else oracle.spmm_baseline(a, b)
    assert bit_equal(got, want)
    assert max_err(got, oracle.spmm_baseline(a, b)) <= 1.0


def test_sddmm_auto_matches_baseline_kernel():
    rng = np.random.default_rng(102)
    p = random_csr(rng, 600, 600, 8, with_values=False)
    x, y = random_dense(rng, 600, 32), random_dense(rng, 600, 32)
    got = asb.sddmm_auto(p, x, y, asb.ProbeConfig(iters=2), asb.ScheduleContext(device=fixed_dev()))
    assert max_err(got, oracle.sddmm(p, x, y)) <= 1.0


def test_default_gpu_profile_and_real_probe():
    dp = asb.DeviceProfile.gpu(0)
    assert "|cores=" in dp.device_sig and dp.cores >= 100
    assert dp.bw_eff > 1e12 and dp.flops_eff > 1e12
    rng = np.random.default_rng(3)
    a = asb.gen_powerlaw(50000, 50000, 800000, 2.2, 4, 4000, 3)
    b = random_dense(rng, 50000, 64)
    cache = asb.ScheduleCache()
    ctx = asb.ScheduleContext(cache=cache)
    d = asb.decide_spmm(a, b, asb.ProbeConfig(), ctx)
    assert d.source == asb.PROBED and d.baseline_ms > 0 and len(d.candidates) == 3
    # guardrail: whatever was chosen is no slower than alpha * t_b on the sample
    if d.choice is not None:
        assert d.t_star <= 0.95 * d.baseline_ms
    assert cache.size() == 1


def test_probe_with_cold_l2_knob(monkeypatch):
    """AUTOSAGE_PROBE_FLUSH_L2 (default 256 MiB, 0 = off) flushes L2 before
    each timed probe: either way the decide probes every candidate and its
    choice keeps the guardrail."""
    for mib in ("32", "0"):
        _cold_probe(monkeypatch, mib)


def _cold_probe(monkeypatch, mib):
    monkeypatch.setenv("AUTOSAGE_PROBE_FLUSH_L2", mib)
    rng = np.random.default_rng(4)
    a = asb.gen_powerlaw(20000, 20000, 300000, 2.2, 4, 2000, 5)
    b = random_dense(rng, 20000, 64)
    d = asb.decide_spmm(a, b, asb.ProbeConfig(iters=2), asb.ScheduleContext(cache=asb.ScheduleCache()))
    assert d.source == asb.PROBED and d.baseline_ms > 0 and len(d.candidates) == 3
    if d.choice is not None:
        assert d.t_star <= 0.95 * d.baseline_ms


def test_probe_config_validation():
    fx = Fixture()
    ctx = asb.ScheduleContext(device=fx.dev)
    with pytest.raises(asb.InvalidArgument):
        asb.decide_spmm(fx.a, fx.b, asb.ProbeConfig(alpha=1.5), ctx)
    with pytest.raises(asb.InvalidArgument):
        asb.decide_spmm(fx.a, fx.b, asb.ProbeConfig(frac=0.0), ctx)


# ---- attention pipeline (proj/tests/test_attention.cpp) -----------------------------
class Ctx:
    def __init__(self):
        self.cache = asb.ScheduleCache()
        self.cfg = asb.ProbeConfig(iters=2)
        self.ctx = asb.ScheduleContext(device=fixed_dev(), cache=self.cache)


def dense_attention_oracle(p, q, k, v):
    n, fv = p.n_rows, v.shape[1]
    out = np.zeros((n, fv))
    for i in range(n):
        cols = p.row_cols(i)
        if cols.size == 0:
            continue
        s = q[i].astype(np.float64) @ k[cols].astype(np.float64).T
        w = np.exp(s - s.max())
        w /= w.sum()
        out[i] = w @ v[cols].astype(np.float64)
    return out


@pytest.mark.parametrize("fused", [False, True])
def test_attention_identity_passes_v(fused):
    c = Ctx()
    rng = np.random.default_rng(1)
    q, k, v = random_dense(rng, 10, 8), random_dense(rng, 10, 8), random_dense(rng, 10, 5)
    out = asb.csr_attention_forward(identity(10), q, k, v, c.cfg, c.ctx, fused=fused)
    assert out.shape == (10, 5)
    assert np.allclose(out, v, rtol=1e-6, atol=0)


@pytest.mark.parametrize("fused", [False, True])
def test_attention_zero_queries_give_neighbor_means(fused):
    c = Ctx()
    rng = np.random.default_rng(2)
    p = random_csr(rng, 30, 30, 6, with_values=False)
    q = np.zeros((30, 8), np.float32)
    k, v = random_dense(rng, 30, 8), random_dense(rng, 30, 4)
    out = asb.csr_attention_forward(p, q, k, v, c.cfg, c.ctx, fused=fused)
    for i in range(30):
        cols = p.row_cols(i)
        want = v[cols].astype(np.float64).mean(axis=0) if cols.size else np.zeros(4)
        for t in range(4):
            assert close(out[i, t], want[t])


def test_attention_random_patterns_match_dense_oracle():
    c = Ctx()
    rng = np.random.default_rng(3)
    for _ in range(12):
        n = 8 + int(rng.integers(0, 57))
        p = random_csr(rng, n, n, 5, with_values=False)
        q, k, v = random_dense(rng, n, 16), random_dense(rng, n, 16), random_dense(rng, n, 9)
        out = asb.csr_attention_forward(p, q, k, v, c.cfg, c.ctx)
        assert max_err(out, dense_attention_oracle(p, q, k, v)) <= 1.0
        for i in range(n):
            if p.degree(i) == 0:
                assert np.all(out[i] == 0.0)


def test_attention_probe_breakdown_sources():
    c = Ctx()
    rng = np.random.default_rng(6)
    p = random_csr(rng, 60, 60, 6, with_values=False)
    q, k, v = (random_dense(rng, 60, 16) for _ in range(3))
    asb.reset_probe_launch_count()
    cold = asb.attention_probe_breakdown(p, q, k, v, c.cfg, c.ctx)
    assert cold.sddmm_decision.source == asb.PROBED and cold.spmm_decision.source == asb.PROBED
    assert cold.sddmm_decision.key.op == asb.SDDMM and cold.spmm_decision.key.op == asb.SPMM
    assert cold.sddmm_decision.key != cold.spmm_decision.key
    assert asb.probe_launch_count() > 0 and c.cache.size() == 2
    asb.reset_probe_launch_count()
    warm = asb.attention_probe_breakdown(p, q, k, v, c.cfg, c.ctx)
    assert warm.sddmm_decision.source == asb.CACHED and warm.spmm_decision.source == asb.CACHED
    assert asb.probe_launch_count() == 0 and bit_equal(warm.output, cold.output)
    c.ctx.replay = asb.ReplayPolicy(replay_only=True)
    rep = asb.attention_probe_breakdown(p, q, k, v, c.cfg, c.ctx, fused=True)
    assert rep.sddmm_decision.source == asb.REPLAYED and rep.spmm_decision.source == asb.REPLAYED
    assert asb.probe_launch_count() == 0 and bit_equal(rep.output, cold.output)


def test_attention_independent_of_forced_variants(monkeypatch):
    rng = np.random.default_rng(5)
    p = random_csr(rng, 40, 40, 6, with_values=False)
    q, k, v = (random_dense(rng, 40, 16) for _ in range(3))
    base = asb.csr_attention_forward(p, q, k, v, Ctx().cfg, Ctx().ctx)
    monkeypatch.setenv("AUTOSAGE_HUB_T", "4")
    monkeypatch.setenv("AUTOSAGE_FTILE", "32")
    forced = Ctx()
    alt = asb.csr_attention_forward(p, q, k, v, forced.cfg, forced.ctx)
    assert np.all(np.abs(alt - base) <= 1e-6 + 2e-5 * np.abs(base))


def test_attention_rejects_incompatible_operands():
    c = Ctx()
    rng = np.random.default_rng(7)
    p = random_csr(rng, 10, 10, 3, with_values=False)
    q = random_dense(rng, 10, 8)
    with pytest.raises(asb.InvalidArgument):
        asb.csr_attention_forward(p, q, random_dense(rng, 10, 7), random_dense(rng, 10, 4),
                                  c.cfg, c.ctx)
    with pytest.raises(asb.InvalidArgument):
        asb.csr_attention_forward(p, q, random_dense(rng, 10, 8), random_dense(rng, 11, 4),
                                  c.cfg, c.ctx)


# ---- multi-GPU building blocks on one device -------------------------------------------
def test_row_range_shards_reassemble_bit_exact():
    rng = np.random.default_rng(8)
    a = hub_graph(rng, 4000, [3000, 1000], 20)
    b = random_dense(rng, 4000, 64)
    cuts = asb.partition_rows(a.rowptr, 4)
    assert np.array_equal(cuts, oracle.partition_rows(a.rowptr, 4))
    g = asb.Graph.from_csr(a)
    bd = cuda(b)
    v = asb.KernelVariant(asb.SPMM, asb.ROWPARALLEL, 64, 4, True)
    parts = []
    for r in range(4):
        shard = g.row_range(int(cuts[r]), int(cuts[r + 1]))
        parts.append(asb.dispatch(v, shard, bd).output.cpu().numpy())
    assert bit_equal(np.concatenate(parts), oracle.spmm_baseline(a, b))


def test_gpu_model_probe_sample_fills_the_device(monkeypatch):
    """B200 model: the probe sample grows to ~AUTOSAGE_GPU_PROBE_NNZ entries
    (row selection unchanged); reference-model profiles keep the reference
    sample size."""
    import math
    rng = np.random.default_rng(77)
    a = random_csr(rng, 3000, 3000, 20)
    b = random_dense(rng, 3000, 32)
    gpu = asb.DeviceProfile.gpu()
    assert gpu.model == 1
    cfg = asb.ProbeConfig(frac=0.02, min_rows=64, iters=2)
    mean = a.nnz / a.n_rows
    monkeypatch.setenv("AUTOSAGE_GPU_PROBE_NNZ", "20000")
    d = asb.decide_spmm(a, b, cfg, asb.ScheduleContext(device=gpu))
    want = min(a.n_rows, max(64, math.ceil(0.02 * a.n_rows), math.ceil(20000 / mean)))
    assert d.sample_rows == want
    ref = asb.DeviceProfile(gpu.device_sig, gpu.bw_eff, gpu.flops_eff, gpu.cores, 0)
    d0 = asb.decide_spmm(a, b, cfg, asb.ScheduleContext(device=ref))
    assert d0.sample_rows == max(64, math.ceil(0.02 * a.n_rows))


@pytest.mark.parametrize("eager", ["1", "0"])
def test_background_graph_sig_matches_oracle(monkeypatch, eager):
    """graph_sig starts in the background at creation for graphs of >= 1M
    entries (AUTOSAGE_EAGER_SIG=0: computed on first use); either way the key
    is the reference's FNV-1a, for host- and device-created graphs, and a
    graph closed before its hash finished is torn down cleanly."""
    import torch
    monkeypatch.setenv("AUTOSAGE_EAGER_SIG", eager)
    m = asb.gen_powerlaw(60_000, 60_000, 1_500_000, 2.2, 4, 5_000, 9)
    want = oracle.graph_sig(m)
    g = asb.Graph.from_csr(m)
    assert g.sig() == want
    g.close()
    asb.Graph.from_csr(m).close()  # destroyed while the background pass may still run
    import paper_2511_17594_b200.torch_ops as tops
    crow = torch.from_numpy(m.rowptr.astype(np.int64)).cuda()
    col = torch.from_numpy(m.colind.astype(np.int32)).cuda()
    gd = tops._graph(crow, col, m.n_cols)
    assert gd.sig() == want


@pytest.mark.parametrize("fused", [True, False])
def test_attention_heads_batched_equals_single_calls(fused):
    """as_csr_attention_forward_heads: each head bit-identical to the
    single-head call; decisions made once (head 1) from a call-local cache."""
    import torch
    rng = np.random.default_rng(77)
    m = hub_graph(rng, 1200, [1100, 500], 9, with_values=False)
    g = asb.Graph.from_csr(m)
    heads = 4
    qs = [torch.from_numpy(rng.uniform(-1, 1, (1200, 32)).astype(np.float32)).cuda() for _ in range(heads)]
    ks = [torch.from_numpy(rng.uniform(-1, 1, (1200, 32)).astype(np.float32)).cuda() for _ in range(heads)]
    vs = [torch.from_numpy(rng.uniform(-1, 1, (1200, 16)).astype(np.float32)).cuda() for _ in range(heads)]
    asb.reset_probe_launch_count()
    outs = asb.csr_attention_forward_heads(g, qs, ks, vs, fused=fused)
    torch.cuda.synchronize()
    batched_probes = asb.probe_launch_count()
    ctx = asb.ScheduleContext(cache=asb.ScheduleCache())
    asb.reset_probe_launch_count()
    for h in range(heads):
        one = asb.csr_attention_forward(g, qs[h], ks[h], vs[h], ctx=ctx, fused=fused)
        one = one.cpu().numpy() if hasattr(one, "cpu") else one
        assert bit_equal(outs[h].cpu().numpy(), one), h
    assert batched_probes == asb.probe_launch_count() > 0  # one decide per op, as the cached single calls
    g.close()


def test_l2_tile_rule_decides_64_wide_spmm_tiles():
    """B200 scheduler: where B overflows the 96 MB L2 budget but a 64-column
    slice fits, SpMM candidates take f_tile 64 (policy.cpp l2_tile_rule); a
    small B keeps the probe's own pick.  The output is the same bits."""
    import torch
    rng = np.random.default_rng(81)
    n = 300_000
    m = asb.gen_powerlaw(n, n, 3_000_000, 2.2, 4, 3_000, 5)
    g = asb.Graph.from_csr(m)
    b = torch.from_numpy(rng.uniform(-1, 1, (n, 128)).astype(np.float32)).cuda()  # 154 MB
    ctx = asb.ScheduleContext(cache=asb.ScheduleCache())
    d = asb.decide_spmm(g, b, None, ctx)
    assert d.choice is not None and d.choice.f_tile == 64, asb.variant_to_string(d.choice)
    c = asb.spmm_auto(g, b, ctx=ctx).cpu().numpy()
    wide = asb.dispatch(dataclasses.replace(d.choice, f_tile=128), g, b).output.cpu().numpy()
    assert bit_equal(c, wide)  # the rule changes the speed, never the bits
    g.close()
