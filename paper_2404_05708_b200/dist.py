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


# ---------------------------------------------------------------------------
# Self all-pairs matrix on W GPUs.  δ is symmetric,
# so only the upper triangle b ≥ a is evaluated.  Rank r owns the rows
# [r0, r1) and computes their columns [r0, n): its diagonal block with
# ffd_cdist_self (each unordered pair once) and the block right of it with
# ffd_cdist.  Row boundaries balance the upper-triangle work Σ_a (n − a) across
# ranks; blocks are padded to one height H so that a single all_gather suffices;
# the lower triangle is then the transpose of the upper one (selection only:
# bit-identical to the single-GPU matrix).
# ---------------------------------------------------------------------------
def self_row_ranges(n: int, world: int) -> list[tuple[int, int]]:
    """Row shards [r0, r1) of the upper-triangle work, one per rank (contiguous,
    covering [0, n), balanced by Σ_a (n − a))."""
    if world < 1:
        raise ValueError("bad world")
    total = n * (n + 1) // 2
    bounds = [0]
    acc, a = 0, 0
    for r in range(1, world):
        target = total * r // world
        while a < n and acc + (n - a) <= target:
            acc += n - a
            a += 1
        bounds.append(a)
    bounds.append(n)
    return [(bounds[r], bounds[r + 1]) for r in range(world)]


def assemble_upper(block, n: int, ranges, group=None):
    """All-gather padded row blocks [H, n] holding the upper-triangle rows of every
    rank (columns < r0 are zero) and mirror them into the full [n, n] matrix."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    H, _ = block.shape
    full = torch.empty((world * H, n), dtype=block.dtype, device=block.device)
    dist.all_gather_into_tensor(full, block.contiguous(), group=group)
    rows = torch.cat([torch.arange(r * H, r * H + (r1 - r0), device=block.device)
                      for r, (r0, r1) in enumerate(ranges)])
    upper = torch.triu(full[rows])
    return upper + torch.triu(upper, diagonal=1).T


def cdist_self(A, norm: str = "l2", group=None):
    """All-pairs δ_dF of the set A against itself over the ranks of `group` (or the
    single local GPU): about half the work of cdist(A, A)."""
    import torch
    import torch.distributed as dist

    import paper_2404_05708_b200 as ffd

    n = A.shape[0]
    if group is None and not (dist.is_available() and dist.is_initialized()):
        return ffd.cdist_self(A, norm=norm)
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    ranges = self_row_ranges(n, world)
    H = max(1, max(r1 - r0 for r0, r1 in ranges))
    r0, r1 = ranges[rank]
    block = torch.zeros((H, n), dtype=torch.float32, device=A.device)
    if r1 > r0:
        block[: r1 - r0, r0:r1] = ffd.cdist_self(A[r0:r1].contiguous(), norm=norm)
        if r1 < n:
            block[: r1 - r0, r1:] = ffd.cdist(A[r0:r1].contiguous(), A[r1:].contiguous(), norm=norm)
    return assemble_upper(block, n, ranges, group)
