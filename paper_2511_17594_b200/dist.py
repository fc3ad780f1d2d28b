"""Row sharding for multi-GPU SpMM / SDDMM / attention.

One process per GPU (torch.distributed over NCCL on B200s, gloo for CPU
tests).  Rows are split into contiguous nnz-balanced ranges
(as_partition_rows: cut_k = lower_bound(rowptr, floor(k*nnz/g))), which is
integer-deterministic, so the concatenated per-rank outputs are bit-identical
to the single-GPU result (every output row is computed by exactly one rank
with the same arithmetic).  The only exchange is an all-gather of the dense
operand's row shards (B for SpMM, Y for SDDMM, K/V for attention): for a
square graph rank r owns rows [cut_r, cut_{r+1}) of every node-feature
matrix.  Shards are padded to the largest shard for all_gather_into_tensor.

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
