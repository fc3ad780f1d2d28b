"""Row sharding for multi-GPU SpMM / SDDMM / attention.

One process per GPU (torch.distributed over NCCL on B200s, gloo for CPU
tests).  Rows are split into contiguous nnz-balanced ranges
(as_partition_rows: cut_k = lower_bound(rowptr, floor(k*nnz/g))), which is
integer-deterministic, so the concatenated per-rank outputs are bit-identical
to the single-GPU result (every output row is computed by exactly one rank
with the same arithmetic).  The only exchange is an all-gather of the dense
operand's row shards (B for SpMM, Y for SDDMM, K/V for attention -- all
heads' K and V in one collective, allgather_heads): for a
square graph rank r owns rows [cut_r, cut_{r+1}) of every node-feature
matrix.  Shards are padded to the largest shard for all_gather_into_tensor.

Overlapped form (blocked_spmm): B's shards travel as one broadcast per owner
and the rank's SpMM consumes them in ascending column blocks as they land
(as_spmm_blocked_*: every row / hub piece carries its f64 accumulator across
blocks, so the product stays bit-identical; tests/test_multiproc.py proves
the exchange with the blocked restatement in the oracle, tests/
test_gpu_blocked.py the kernels).

Padded-native layout (what bench.py runs): each rank's shard graph has its
column indices remapped once, c -> owner(c) * shard + (c - cut[owner(c)]),
so the kernels gather straight from the padded all-gather buffer -- no
per-step un-pad copy, and the rank's own rows are the all-gather input
in place.  The remap is monotone in c, so every row keeps its entry order
and the results stay bit-identical.  allgather_rows (un-padded, global row
order) remains for callers that need the plain matrix.
"""
from __future__ import annotations

import numpy as np

from . import CsrMatrix, partition_rows


def row_range_host(m: CsrMatrix, r0: int, r1: int) -> CsrMatrix:
    """Rows [r0, r1) of a host CSR with rebased rowptr and global columns."""
    e0, e1 = int(m.rowptr[r0]), int(m.rowptr[r1])
    rp = (m.rowptr[r0:r1 + 1] - np.uint64(e0)).astype(np.uint64)
    return CsrMatrix(r1 - r0, m.n_cols, rp, m.colind[e0:e1],
                     None if m.val is None else m.val[e0:e1])


class RowSharding:
    """Rank r's view of an nnz-balanced row partition of an n-row graph."""

    def __init__(self, rowptr, world: int, rank: int):
        self.world, self.rank = world, rank
        self.cuts = partition_rows(rowptr, world)
        self.r0, self.r1 = int(self.cuts[rank]), int(self.cuts[rank + 1])
        self.sizes = np.diff(self.cuts.astype(np.int64))
        self.shard = int(self.sizes.max()) if world else 0
        self.n = int(self.cuts[-1])
        # padded all-gather position of global row i
        self.perm = np.concatenate([r * self.shard + np.arange(self.sizes[r])
                                    for r in range(world)]).astype(np.int64)
        self._perm_t = {}

    def remap_cols(self, colind) -> np.ndarray:
        """Global column -> position in the padded all-gather buffer."""
        c = np.asarray(colind, dtype=np.int64)
        owner = np.searchsorted(self.cuts.astype(np.int64), c, side="right") - 1
        return (owner * self.shard + (c - self.cuts.astype(np.int64)[owner])).astype(np.uint32)

    @property
    def padded_rows(self) -> int:
        return self.world * self.shard

    def shard_graph_host(self, m: CsrMatrix) -> CsrMatrix:
        """This rank's rows with columns remapped into the padded layout."""
        part = row_range_host(m, self.r0, self.r1)
        if self.world == 1:
            return part
        return CsrMatrix(part.n_rows, self.padded_rows, part.rowptr, self.remap_cols(part.colind), part.val)

    def allgather_padded(self, local_padded, out_padded, group=None, async_op=False):
        """All-gather (shard x F) padded row blocks into (world*shard x F);
        returns the work handle when async_op."""
        import torch.distributed as dist
        if dist.get_backend(group) == "nccl":
            return dist.all_gather_into_tensor(out_padded, local_padded, group=group, async_op=async_op)
        return dist.all_gather(list(out_padded.split(self.shard)), local_padded, group=group,
                               async_op=async_op)

    def column_cuts(self, groups: int = 0) -> np.ndarray:
        """Column cuts of the padded all-gather layout by owner groups: block
        k holds the columns (B rows) of ranks [k*per, (k+1)*per), per =
        ceil(world / groups); groups 0 = one block per rank.  Ascending
        blocks are ascending global columns, so a blocked SpMM over them
        keeps every row's CSR order (as_spmm_blocked_*)."""
        g = groups if groups and groups > 0 else self.world
        per = -(-self.world // g)
        owners = list(range(0, self.world, per)) + [self.world]
        return np.asarray([o * self.shard for o in owners], dtype=np.uint64)

    def owners_of_block(self, k: int, groups: int = 0):
        g = groups if groups and groups > 0 else self.world
        per = -(-self.world // g)
        return list(range(k * per, min(self.world, (k + 1) * per)))

    def broadcast_shards(self, local_padded, out_padded, group=None):
        """The all-gather as one async broadcast per owner, in rank order,
        straight into its slice of the padded buffer: returns the work
        handles, so a consumer waits only for the shards it needs next
        (NCCL: handle.wait() orders the current stream after the copy)."""
        import torch.distributed as dist
        handles = []
        for r in range(self.world):
            dst = out_padded[r * self.shard:(r + 1) * self.shard]
            if r == self.rank:
                dst.copy_(local_padded)
            handles.append(dist.broadcast(dst, src=r, group=group, async_op=True))
        return handles

    def blocked_spmm(self, local_padded, out_padded, run_block, groups: int = 0, group=None):
        """Exchange B's row shards and consume them as they land: block k's
        SpMM (run_block(k)) starts once its owners' shards are in, while the
        later shards are still in flight."""
        handles = self.broadcast_shards(local_padded, out_padded, group=group)
        n_blocks = self.column_cuts(groups).size - 1
        for k in range(n_blocks):
            for r in self.owners_of_block(k, groups):
                handles[r].wait()
            run_block(k)

    def allgather_heads(self, local_heads, group=None):
        """K / V of all heads in ONE collective: local (H, shard, F) -> the
        per-head padded operands (H, world*shard, F), each head contiguous
        (one all-gather, then one device-side reshuffle of the
        (world, H, shard, F) result)."""
        import torch
        import torch.distributed as dist
        h, shard, f = local_heads.shape
        gathered = torch.empty((self.world, h, shard, f), dtype=local_heads.dtype, device=local_heads.device)
        if dist.get_backend(group) == "nccl":
            dist.all_gather_into_tensor(gathered, local_heads.contiguous(), group=group)
        else:
            dist.all_gather(list(gathered.unbind(0)), local_heads.contiguous(), group=group)
        return gathered.permute(1, 0, 2, 3).reshape(h, self.world * shard, f)

    def pad_heads(self, full_heads_local_rows):
        """(H, local_rows, F) -> (H, shard, F) zero-padded all-gather input."""
        import torch
        h, n, f = full_heads_local_rows.shape
        out = torch.zeros((h, self.shard, f), dtype=full_heads_local_rows.dtype,
                          device=full_heads_local_rows.device)
        out[:, :n] = full_heads_local_rows
        return out

    @property
    def local_rows(self) -> int:
        return self.r1 - self.r0

    def _perm(self, device):
        import torch
        key = str(device)
        if key not in self._perm_t:
            self._perm_t[key] = torch.from_numpy(self.perm).to(device)
        return self._perm_t[key]

    def allgather_rows(self, local, group=None, out_padded=None):
        """All-gather the ranks' row shards of a dense (rows x F) matrix and
        return the full n x F matrix in global row order."""
        import torch
        import torch.distributed as dist
        f = local.shape[1]
        if self.world == 1:
            return local
        padded = torch.zeros((self.shard, f), dtype=local.dtype, device=local.device)
        padded[: local.shape[0]] = local
        if out_padded is None:
            out_padded = torch.empty((self.world * self.shard, f), dtype=local.dtype,
                                     device=local.device)
        if dist.get_backend(group) == "nccl":
            dist.all_gather_into_tensor(out_padded, padded, group=group)
        else:  # gloo: list form
            parts = list(out_padded.split(self.shard))
            dist.all_gather(parts, padded, group=group)
        return out_padded.index_select(0, self._perm(local.device))
