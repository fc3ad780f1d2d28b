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


def _worker_blocked(rank, world, port, results):
    """B's shards broadcast per owner and consumed block by block as they
    land (RowSharding.blocked_spmm), each block's arithmetic the oracle's
    restatement of as_spmm_blocked_* (segment accumulators carried across
    ascending column blocks): the concatenated rows equal the single-process
    SpMM, rowparallel and hubsplit, bit for bit."""
    import oracle
    import paper_2511_17594_b200 as asb
    from paper_2511_17594_b200.dist import RowSharding
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        m = asb.gen_powerlaw(4000, 4000, 120000, 2.0, 3, 3500, 17)
        f = 20
        b = asb.fill_uniform(m.n_cols * f, 7, (m.n_cols, f))
        sh = RowSharding(m.rowptr, world, rank)
        pg = sh.shard_graph_host(m)
        loc = torch.zeros((sh.shard, f))
        loc[: sh.local_rows] = torch.from_numpy(b[sh.r0:sh.r1])
        ok = True
        for groups in (0, 1, world):
            for hub_t in (0, 64):
                pad = torch.full((sh.padded_rows, f), float("nan"))
                cuts = sh.column_cuts(groups)
                landed = []

                def run_block(k):
                    # block k may read only the shards of its owners, landed now
                    for r in sh.owners_of_block(k, groups):
                        landed.append(r)
                sh.blocked_spmm(loc, pad, run_block, groups=groups)
                c = oracle.spmm_blocked(pg, pad.numpy(), cuts, hub_t)
                want = (oracle.spmm_hubsplit(m, b, hub_t) if hub_t else oracle.spmm_baseline(m, b))[sh.r0:sh.r1]
                ok = ok and landed == list(range(world)) and np.array_equal(c.view(np.uint32), want.view(np.uint32))
        flags = torch.tensor([1 if ok else 0])
        dist.all_reduce(flags, op=dist.ReduceOp.MIN)
        if rank == 0:
            results["blocked"] = bool(flags.item() == 1)
    finally:
        dist.destroy_process_group()


def _worker_heads(rank, world, port, results):
    """c5-style sharded attention: K and V of all heads gathered in one
    collective (allgather_heads), each head's attention on the rank's rows
    over the padded layout; equals the single-process attention rows."""
    import oracle
    import paper_2511_17594_b200 as asb
    from paper_2511_17594_b200.dist import RowSharding
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        m = asb.gen_powerlaw(2500, 2500, 50000, 2.2, 3, 2000, 23, with_values=False)
        heads, f = 3, 16
        q = [asb.fill_uniform(m.n_rows * f, 1 + 3 * h, (m.n_rows, f)) for h in range(heads)]
        k = [asb.fill_uniform(m.n_cols * f, 2 + 3 * h, (m.n_cols, f)) for h in range(heads)]
        v = [asb.fill_uniform(m.n_cols * f, 3 + 3 * h, (m.n_cols, f)) for h in range(heads)]
        sh = RowSharding(m.rowptr, world, rank)
        pg = sh.shard_graph_host(m)
        k_loc = sh.pad_heads(torch.from_numpy(np.stack([kk[sh.r0:sh.r1] for kk in k])))
        v_loc = sh.pad_heads(torch.from_numpy(np.stack([vv[sh.r0:sh.r1] for vv in v])))
        kg, vg = sh.allgather_heads(k_loc), sh.allgather_heads(v_loc)  # one collective each
        ok = True
        for h in range(heads):
            got = oracle.attention(pg, q[h][sh.r0:sh.r1], kg[h].numpy(), vg[h].numpy())
            want = oracle.attention(m, q[h], k[h], v[h])[sh.r0:sh.r1]
            ok = ok and np.array_equal(got.view(np.uint32), want.view(np.uint32))
        flags = torch.tensor([1 if ok else 0])
        dist.all_reduce(flags, op=dist.ReduceOp.MIN)
        if rank == 0:
            results["heads"] = bool(flags.item() == 1)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("worker,key", [(_worker_blocked, "blocked"), (_worker_heads, "heads")])
def test_overlapped_exchanges_world2(worker, key):
    ctx = mp.get_context("spawn")
    manager = ctx.Manager()
    results = manager.dict()
    port = _free_port()
    procs = [ctx.Process(target=worker, args=(r, 2, port, results)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=240)
        assert p.exitcode == 0
    assert results.get(key)


def test_bench_spawns_ranks_itself():
    """`bench.py --gpus 2` outside torchrun re-launches under
    torch.distributed.run (the reference arm needs no GPU: rank 0 prints the
    line, rank 1 exits)."""
    import json
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    env["PYTHONPATH"] = root
    r = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--impl", "reference", "--gpus", "2",
                        "--config", "c1", "--steps", "1", "--warmup", "3"], cwd=root, env=env,
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["n_gpus"] == 2 and d["value"] > 0
