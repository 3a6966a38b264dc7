"""Multi-GPU all-pairs distances: row shards of A per rank + one all-gather.

ffd_cdist is embarrassingly parallel over output rows: rank r
computes rows [r·⌈nA/W⌉, (r+1)·⌈nA/W⌉) of the [nA, nB] matrix against all of B
(B is replicated, 20 MB for config 4), then one
``all_gather_into_tensor`` over NCCL (NVLink 5 / NVSwitch) assembles the full
matrix on every rank.  The gather is the only collective; blocks are padded to
equal height so a single all-gather suffices, and the result is identical bit
for bit for any world size (δ only selects values).
"""
from __future__ import annotations

import math


def row_range(n_rows: int, world: int, rank: int) -> tuple[int, int, int]:
    """(row_begin, row_end, block_rows) of `rank`'s shard; block_rows is the padded
    common block height (⌈n_rows / world⌉)."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError("bad world/rank")
    blk = max(1, math.ceil(n_rows / world))
    r0 = min(n_rows, rank * blk)
    r1 = min(n_rows, r0 + blk)
    return r0, r1, blk


def assemble(block, n_rows: int, group=None):
    """All-gather equal-height row blocks [blk, nB] of every rank into [n_rows, nB]."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    blk, nB = block.shape
    full = torch.empty((world * blk, nB), dtype=block.dtype, device=block.device)
    dist.all_gather_into_tensor(full, block.contiguous(), group=group)
    return full[:n_rows]


def cdist(A, B, norm: str = "l2", group=None, return_block: bool = False):
    """All-pairs δ_dF over the ranks of `group` (or the single local GPU).

    A [nA, lenA, dim], B [nB, lenB, dim] CUDA tensors, identical on every rank.
    Returns the full [nA, nB] matrix on every rank (or only this rank's block
    with return_block=True, skipping the collective)."""
    import torch
    import torch.distributed as dist

    import paper_2404_05708_b200 as ffd

    nA, nB = A.shape[0], B.shape[0]
    if group is None and not (dist.is_available() and dist.is_initialized()):
        return ffd.cdist(A, B, norm=norm)
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    r0, r1, blk = row_range(nA, world, rank)
    block = torch.empty((blk, nB), dtype=torch.int64 if A.dtype == torch.int32 else torch.float32,
                        device=A.device)
    if r1 > r0:
        ffd.cdist(A, B, norm=norm, rows=(r0, r1), out=block)
    if return_block:
        return block[: r1 - r0], (r0, r1)
    return assemble(block, nA, group)
