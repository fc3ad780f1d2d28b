"""World-size-2 multi-process test of the row-sharded path on CPU (gloo).

Each rank takes its nnz-balanced row range (paper_2511_17594_b200.dist),
all-gathers the dense operand's row shards exactly as bench.py does over
NCCL, and computes its rows; the concatenation must equal the single-process
result bit for bit.  The per-rank arithmetic here is the CPU oracle (the
checker) because this machine has no GPU; on B200s the same sharding feeds
the sm_100a kernels (tests/test_gpu_scheduler.py covers the per-shard GPU
kernels against the same concatenation property).
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, results):
    import oracle
    import paper_2511_17594_b200 as asb
    from paper_2511_17594_b200.dist import RowSharding, row_range_host
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        m = asb.gen_powerlaw(3000, 3000, 60000, 2.0, 3, 2500, 11)
        f = 24
        b = asb.fill_uniform(m.n_cols * f, 5, (m.n_cols, f))
        x = asb.fill_uniform(m.n_rows * f, 6, (m.n_rows, f))
        sh = RowSharding(m.rowptr, world, rank)
        local_b = torch.from_numpy(b[sh.r0:sh.r1].copy())
        full_b = sh.allgather_rows(local_b).numpy()
        assert np.array_equal(full_b, b)
        part = row_range_host(m, sh.r0, sh.r1)
        c_local = torch.from_numpy(oracle.spmm_baseline(part, full_b))
        s_local = torch.from_numpy(oracle.sddmm(part, x[sh.r0:sh.r1], full_b, 64, True))
        # gather outputs (row-sharded C, nnz-sharded SDDMM values) to every rank
        c_full = sh.allgather_rows(c_local).numpy()
        lens = [int(m.rowptr[sh.cuts[r + 1]] - m.rowptr[sh.cuts[r]]) for r in range(world)]
        pad = max(lens)
        sp = torch.zeros(pad)
        sp[: s_local.numel()] = s_local
        parts = [torch.empty(pad) for _ in range(world)]
        dist.all_gather(parts, sp)
        s_full = np.concatenate([p[:n].numpy() for p, n in zip(parts, lens)])
        # padded-native layout (bench.py): remapped shard graph over the padded
        # all-gather buffer, no un-pad copy -- same bits
        loc_pad = torch.zeros((sh.shard, f))
        loc_pad[: sh.local_rows] = local_b
        out_pad = torch.empty((sh.padded_rows, f))
        sh.allgather_padded(loc_pad, out_pad)
        pg = sh.shard_graph_host(m)
        assert pg.n_cols == world * sh.shard and asb.validate(pg) is None
        c_pad = oracle.spmm_baseline(pg, out_pad.numpy())
        s_pad = oracle.sddmm(pg, x[sh.r0:sh.r1], out_pad.numpy(), 64, True)
        same_pad = (np.array_equal(c_pad.view(np.uint32), c_local.numpy().view(np.uint32)) and
                    np.array_equal(s_pad.view(np.uint32), s_local.numpy().view(np.uint32)))
        flags = torch.tensor([1 if same_pad else 0])
        dist.all_reduce(flags, op=dist.ReduceOp.MIN)
        if rank == 0:
            want_c = oracle.spmm_baseline(m, b)
            want_s = oracle.sddmm(m, x, b, 64, True)
            results["padded"] = bool(flags.item() == 1)
            results["spmm"] = bool(np.array_equal(c_full.view(np.uint32), want_c.view(np.uint32)))
            results["sddmm"] = bool(np.array_equal(s_full.view(np.uint32), want_s.view(np.uint32)))
            results["balanced"] = max(lens) - m.nnz / world <= int(m.degrees().max())
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_row_sharded_spmm_sddmm_concatenate_bit_exact(world):
    ctx = mp.get_context("spawn")
    manager = ctx.Manager()
    results = manager.dict()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, results)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=240)
        assert p.exitcode == 0
    assert results.get("spmm") and results.get("sddmm") and results.get("balanced")
    assert results.get("padded")
