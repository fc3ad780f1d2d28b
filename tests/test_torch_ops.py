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
    for name in ("spmm_csr", "spmm_csr_auto", "sddmm_csr", "csr_attention"):
        assert hasattr(torch.ops.autosage, name)
    with FakeTensorMode():
        crow = torch.empty(11, dtype=torch.int64)
        col = torch.empty(30, dtype=torch.int32)
        val = torch.empty(30)
        b = torch.empty(7, 16)
        assert torch.ops.autosage.spmm_csr(crow, col, val, b, "").shape == (10, 16)
        assert torch.ops.autosage.sddmm_csr(crow, col, torch.empty(10, 16), b, "").shape == (30,)
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
def test_attention_op_matches_library_path():
    rng = np.random.default_rng(62)
    a = hub_graph(rng, 500, [450], 6, with_values=False)
    crow, col, _ = _csr(a)
    q, k, v = (torch.from_numpy(random_dense(rng, 500, 32)).cuda() for _ in range(3))
    got = torch.ops.autosage.csr_attention(crow, col, q, k, v, False)
    want = asb.csr_attention_forward(a, q, k, v)
    assert bit_equal(got.cpu().numpy(), want.cpu().numpy() if hasattr(want, "cpu") else want)
