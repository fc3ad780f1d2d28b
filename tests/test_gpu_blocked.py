"""Column-blocked SpMM kernels (as_spmm_blocked_*, csrc/spmm_blocked.cu):
consuming B one column block at a time, with every row / hub piece carrying
its f64 accumulator across blocks, reproduces the unblocked SpMM -- and so
the reference (src/kernels.cpp:210-334) -- bit for bit, for any cuts
(empty blocks, single-column blocks, a hub split across all blocks), every
mapping, vector and scalar tiles, values, pattern-only and value overrides."""
import numpy as np
import pytest
import torch

import oracle
import paper_2511_17594_b200 as asb
from tests.util import bit_equal, cuda, hub_graph, n_bit_diff, random_dense

pytestmark = pytest.mark.gpu

SP, RP, HS = asb.SPMM, asb.ROWPARALLEL, asb.HUBSPLIT


def run_blocked(g, variant, cuts, b, vals=None):
    p = asb.BlockedSpmm(g, variant, cuts)
    c = torch.full((g.n_rows, b.shape[1]), float("nan"), device="cuda")
    for k in range(p.n_blocks):
        p.run(k, b, c, vals=vals)
    torch.cuda.synchronize()
    p.close()
    return c.cpu().numpy()


@pytest.mark.parametrize("f", [16, 33, 64, 128])
def test_blocked_equals_unblocked_for_any_cuts(f):
    rng = np.random.default_rng(40 + f)
    a = hub_graph(rng, 5000, [4900, 4200, 2049, 700, 300], 12)
    b = random_dense(rng, 5000, f)
    g = asb.Graph.from_csr(a)
    bd = cuda(b)
    cut_sets = [[0, 5000], [0, 2500, 5000], [0, 0, 1, 1000, 1000, 4999, 5000],
                list(np.sort(rng.choice(np.arange(1, 5000), 7, replace=False))) ]
    cut_sets[-1] = [0] + cut_sets[-1] + [5000]
    for variant, want in ((None, oracle.spmm_baseline(a, b)),
                          (asb.KernelVariant(SP, RP, 64, 1, True), oracle.spmm_baseline(a, b)),
                          (asb.KernelVariant(SP, HS, 64, 1, True, 256), oracle.spmm_hubsplit(a, b, 256)),
                          (asb.KernelVariant(SP, HS, 32, 4, False, 1), oracle.spmm_hubsplit(a, b, 1))):
        for cuts in cut_sets:
            got = run_blocked(g, variant, cuts, bd)
            assert bit_equal(got, want), (variant, cuts, n_bit_diff(got, want))
            assert bit_equal(got, oracle.spmm_blocked(a, b, cuts, variant.hub_threshold if variant is not None
                                                      and variant.mapping == HS else 0))


def test_blocked_pattern_only_values_override_and_reuse():
    rng = np.random.default_rng(77)
    a = hub_graph(rng, 3000, [2500, 600], 9, with_values=False)
    b = random_dense(rng, 3000, 64)
    g = asb.Graph.from_csr(a)
    bd = cuda(b)
    cuts = [0, 700, 1400, 3000]
    assert bit_equal(run_blocked(g, None, cuts, bd), oracle.spmm_baseline(a, b))
    w = rng.uniform(-1, 1, a.nnz).astype(np.float32)
    aw = asb.CsrMatrix(a.n_rows, a.n_cols, a.rowptr, a.colind, w)
    hv = asb.KernelVariant(SP, HS, 64, 1, True, 256)
    p = asb.BlockedSpmm(g, hv, cuts)
    c = torch.empty((3000, 64), device="cuda")
    for _ in range(2):  # a plan runs any number of products
        for k in range(p.n_blocks):
            p.run(k, bd, c, vals=cuda(w))
        torch.cuda.synchronize()
        assert bit_equal(c.cpu().numpy(), oracle.spmm_hubsplit(aw, b, 256))
    p.close()


def test_blocked_plan_validation():
    rng = np.random.default_rng(78)
    a = hub_graph(rng, 100, [50], 3)
    g = asb.Graph.from_csr(a)
    with pytest.raises(asb.InvalidArgument):
        asb.BlockedSpmm(g, None, [0, 50])  # does not reach n_cols
    with pytest.raises(asb.InvalidArgument):
        asb.BlockedSpmm(g, None, [0, 60, 40, 100])  # decreasing
    p = asb.BlockedSpmm(g, None, [0, 50, 100])
    with pytest.raises(asb.InvalidArgument):
        p.run(2, cuda(random_dense(rng, 100, 8)), torch.empty((100, 8), device="cuda"))
