"""torch.ops.autosage.* (paper_2511_17594_b200/torch_ops.py):
registration and fake (meta) shapes on CPU; bit-exact results on the GPU."""
import numpy as np
import pytest
import torch

import oracle
import paper_2511_17594_b200 as asb
import paper_2511_17594_b200.torch_ops  # noqa: F401  (registers the ops)
from tests.util import bit_equal, hub_graph, random_dense


def test_ops_are_registered_with_fake_shapes():
    from torch._subclasses.fake_tensor import FakeTensorMode
    for name in ("spmm_csr", "spmm_csr_split", "spmm_csr_auto", "sddmm_csr", "sddmm_csr_auto", "csr_attention"):
        assert hasattr(torch.ops.autosage, name)
    with FakeTensorMode():
        crow = torch.empty(11, dtype=torch.int64)
        col = torch.empty(30, dtype=torch.int32)
        val = torch.empty(30)
        b = torch.empty(7, 16)
        assert torch.ops.autosage.spmm_csr(crow, col, val, b, "").shape == (10, 16)
        assert torch.ops.autosage.sddmm_csr(crow, col, torch.empty(10, 16), b, "").shape == (30,)
        assert torch.ops.autosage.spmm_csr_split(crow, col, val, b, 256, 64, True).shape == (10, 16)
        assert torch.ops.autosage.sddmm_csr_auto(crow, col, torch.empty(10, 16), b).shape == (30,)
        assert torch.ops.autosage.csr_attention(crow, col, torch.empty(10, 16), b, torch.empty(7, 8),
                                                False).shape == (10, 8)


def _csr(m):
    return (torch.from_numpy(m.rowptr.astype(np.int64)).cuda(), torch.from_numpy(m.colind.astype(np.int32)).cuda(),
            torch.from_numpy(m.val).cuda() if m.val is not None else torch.empty(0, device="cuda"))


@pytest.mark.gpu
def test_spmm_and_sddmm_ops_bit_exact():
    rng = np.random.default_rng(61)
    a = hub_graph(rng, 900, [800, 300], 7)
    crow, col, val = _csr(a)
    b = random_dense(rng, 900, 64)
    bt = torch.from_numpy(b).cuda()
    want = oracle.spmm_baseline(a, b)
    for v in ("", "spmm:rowparallel:ft=64:rpc=4:vec=1:hubt=256"):
        assert bit_equal(torch.ops.autosage.spmm_csr(crow, col, val, bt, v).cpu().numpy(), want)
    assert bit_equal(torch.ops.autosage.spmm_csr(crow, col, val, bt, "spmm:hubsplit:ft=32:rpc=4:vec=0:hubt=64")
                     .cpu().numpy(), oracle.spmm_hubsplit(a, b, 64))
    auto = torch.ops.autosage.spmm_csr_auto(crow, col, val, bt).cpu().numpy()
    assert bit_equal(auto, want) or bit_equal(auto, oracle.spmm_hubsplit(a, b, 256))
    x = random_dense(rng, 900, 32)
    y = random_dense(rng, 900, 32)
    got = torch.ops.autosage.sddmm_csr(crow, col, torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda(),
                                       "sddmm:rowparallel:ft=32:rpc=4:vec=1:hubt=256")
    assert bit_equal(got.cpu().numpy(), oracle.sddmm(a, x, y, 32, True))


@pytest.mark.gpu
def test_split_and_sddmm_auto_ops_bit_exact_with_grads():
    """spmm_csr_split (the paper's split SpMM) and sddmm_csr_auto
    (PAPER.md:286): forward bit-exact against the oracle at several hub
    thresholds, and gradients through the same backward as spmm_csr /
    sddmm_csr."""
    rng = np.random.default_rng(64)
    a = hub_graph(rng, 900, [850, 400, 300], 9)
    crow, col, val = _csr(a)
    b = random_dense(rng, 900, 48)
    for hub_t, ft, vec in ((1, 64, True), (64, 32, False), (256, 0, True), (5000, 64, True)):
        bt = torch.from_numpy(b).cuda().requires_grad_(True)
        c = torch.ops.autosage.spmm_csr_split(crow, col, val, bt, hub_t, ft, vec)
        assert bit_equal(c.detach().cpu().numpy(), oracle.spmm_hubsplit(a, b, hub_t)), (hub_t, ft, vec)
        c.sum().backward()
        ref = torch.from_numpy(b).cuda().requires_grad_(True)
        torch.ops.autosage.spmm_csr(crow, col, val, ref, "").sum().backward()
        assert bit_equal(bt.grad.cpu().numpy(), ref.grad.cpu().numpy()), hub_t
    with pytest.raises(ValueError):
        torch.ops.autosage.spmm_csr_split(crow, col, val, torch.from_numpy(b).cuda(), 0, 64, True)
    x = torch.from_numpy(random_dense(rng, 900, 32)).cuda().requires_grad_(True)
    y = torch.from_numpy(random_dense(rng, 900, 32)).cuda().requires_grad_(True)
    s = torch.ops.autosage.sddmm_csr_auto(crow, col, x, y)
    xs, ys = x.detach().cpu().numpy(), y.detach().cpu().numpy()
    got = s.detach().cpu().numpy()
    assert bit_equal(got, oracle.sddmm(a, xs, ys)) or any(
        bit_equal(got, oracle.sddmm(a, xs, ys, ft, True)) for ft in (32, 64, 128))
    s.sum().backward()
    x2, y2 = (t.detach().clone().requires_grad_(True) for t in (x, y))
    torch.ops.autosage.sddmm_csr(crow, col, x2, y2, "").sum().backward()
    assert bit_equal(x.grad.cpu().numpy(), x2.grad.cpu().numpy())
    assert bit_equal(y.grad.cpu().numpy(), y2.grad.cpu().numpy())


@pytest.mark.gpu
def test_attention_op_matches_library_path():
    rng = np.random.default_rng(62)
    a = hub_graph(rng, 500, [450], 6, with_values=False)
    crow, col, _ = _csr(a)
    q, k, v = (torch.from_numpy(random_dense(rng, 500, 32)).cuda() for _ in range(3))
    got = torch.ops.autosage.csr_attention(crow, col, q, k, v, False)
    want = asb.csr_attention_forward(a, q, k, v)
    assert bit_equal(got.cpu().numpy(), want.cpu().numpy() if hasattr(want, "cpu") else want)


@pytest.mark.gpu
def test_graph_cache_survives_address_reuse_and_weight_updates():
    """a freed CSR's addresses reused by a different graph must not
    hit the stale cached graph; updating the weights in place must take
    effect without rebuilding the structure."""
    rng = np.random.default_rng(63)
    b = random_dense(rng, 400, 32)
    bt = torch.from_numpy(b).cuda()
    for trial in range(4):
        a = hub_graph(rng, 400, [300 - trial], 5 + trial)
        crow, col, val = _csr(a)
        got = torch.ops.autosage.spmm_csr(crow, col, val, bt, "").cpu().numpy()
        assert bit_equal(got, oracle.spmm_baseline(a, b)), trial
        del crow, col, val  # the next trial's tensors may land on the same addresses
    a = hub_graph(rng, 400, [350], 9)
    crow, col, val = _csr(a)
    torch.ops.autosage.spmm_csr(crow, col, val, bt, "")
    val.mul_(0.5)  # in place: same storage, new weights
    w = a.val * np.float32(0.5)
    want = oracle.spmm_baseline(asb.CsrMatrix(a.n_rows, a.n_cols, a.rowptr, a.colind, w), b)
    assert bit_equal(torch.ops.autosage.spmm_csr(crow, col, val, bt, "").cpu().numpy(), want)
    assert bit_equal(torch.ops.autosage.spmm_csr_auto(crow, col, val, bt).cpu().numpy(), want) or \
        bit_equal(torch.ops.autosage.spmm_csr_auto(crow, col, val, bt).cpu().numpy(),
                  oracle.spmm_hubsplit(asb.CsrMatrix(a.n_rows, a.n_cols, a.rowptr, a.colind, w), b, 256))


@pytest.mark.gpu
def test_ops_reject_malformed_operands():
    rng = np.random.default_rng(64)
    a = hub_graph(rng, 200, [150], 4)
    crow, col, val = _csr(a)
    b = torch.from_numpy(random_dense(rng, 200, 16)).cuda()
    with pytest.raises(asb.InvalidArgument):  # a column past the dense operand's rows
        torch.ops.autosage.spmm_csr(crow, col, val, b[:100], "")
    bad = col.clone()
    bad[1], bad[2] = col[2], col[1]  # row 0 (degree 150) out of order
    with pytest.raises(asb.InvalidArgument):
        torch.ops.autosage.spmm_csr(crow, bad, val, b, "")
    x = torch.from_numpy(random_dense(rng, 200, 16)).cuda()
    with pytest.raises(ValueError):  # feature widths differ
        torch.ops.autosage.sddmm_csr(crow, col, x, b[:, :8].contiguous(), "")
    with pytest.raises(ValueError):  # k and v row counts differ
        torch.ops.autosage.csr_attention(crow, col, x, b, b[:150].contiguous(), False)
    with pytest.raises(ValueError):  # weights of the wrong length
        torch.ops.autosage.spmm_csr(crow, col, val[:-1], b, "")


@pytest.mark.gpu
def test_one_graph_from_two_streams_and_threads():
    """operators on one cached graph from different streams and
    threads share its scratch; they must serialise (GraphUse), giving the
    same bits as one stream."""
    import threading
    rng = np.random.default_rng(65)
    a = hub_graph(rng, 3000, [2500, 2100, 900], 30)
    crow, col, val = _csr(a)
    xs = [torch.from_numpy(random_dense(rng, 3000, 64)).cuda() for _ in range(4)]
    want_s = [oracle.sddmm(a, x.cpu().numpy(), x.cpu().numpy(), 64, False) for x in xs]
    want_c = [oracle.spmm_hubsplit(a, x.cpu().numpy(), 64) for x in xs]
    streams = [torch.cuda.Stream() for _ in range(4)]
    outs = [None] * 4
    torch.ops.autosage.spmm_csr(crow, col, val, xs[0], "")  # build + cache the graph first
    torch.cuda.synchronize()

    def work(i):
        with torch.cuda.stream(streams[i]):
            for _ in range(3):
                s = torch.ops.autosage.sddmm_csr(crow, col, xs[i], xs[i], "sddmm:rowparallel:ft=32:rpc=1:vec=0:hubt=256")
                c = torch.ops.autosage.spmm_csr(crow, col, val, xs[i], "spmm:hubsplit:ft=64:rpc=1:vec=1:hubt=64")
            streams[i].synchronize()
            outs[i] = (s.cpu().numpy(), c.cpu().numpy())
    th = [threading.Thread(target=work, args=(i,)) for i in range(4)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    for i in range(4):
        assert bit_equal(outs[i][0], want_s[i]) and bit_equal(outs[i][1], want_c[i]), i


@pytest.mark.gpu
def test_auto_ops_persist_and_replay_the_cache_file(monkeypatch, tmp_path):
    """AUTOSAGE_CACHE: the *_auto ops load the cache file on
    first use and rewrite it when they add a decision; a fresh process-wide
    cache under AUTOSAGE_REPLAY_ONLY + STRICT then replays it without a probe,
    with the same bits."""
    import paper_2511_17594_b200.torch_ops as tops
    rng = np.random.default_rng(65)
    a = hub_graph(rng, 700, [650, 300], 8)
    crow, col, val = _csr(a)
    b = torch.from_numpy(random_dense(rng, 700, 32)).cuda()
    path = tmp_path / "autosage.cache"
    monkeypatch.setenv("AUTOSAGE_CACHE", str(path))
    monkeypatch.setattr(tops, "_CACHE", None)
    first = torch.ops.autosage.spmm_csr_auto(crow, col, val, b).cpu().numpy()
    lines = path.read_text().strip().splitlines()
    assert len(lines) == 1 and "spmm" in lines[0]
    monkeypatch.setattr(tops, "_CACHE", None)
    monkeypatch.setenv("AUTOSAGE_REPLAY_ONLY", "1")
    monkeypatch.setenv("AUTOSAGE_REPLAY_STRICT", "1")
    asb.reset_probe_launch_count()
    again = torch.ops.autosage.spmm_csr_auto(crow, col, val, b).cpu().numpy()
    assert asb.probe_launch_count() == 0
    assert bit_equal(first, again)
    x = torch.from_numpy(random_dense(rng, 700, 16)).cuda()
    with pytest.raises(asb.ReplayMiss):  # no SDDMM decision in the file, strict replay
        torch.ops.autosage.sddmm_csr_auto(crow, col, x, b[:, :16].contiguous())
    monkeypatch.setattr(tops, "_CACHE", None)
