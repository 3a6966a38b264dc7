"""Multi-GPU all-pairs distances: row shards of A per rank, then the matrix on every rank.

ffd_cdist is embarrassingly parallel over output rows (PAPER L259:
the pairs are independent): rank r computes rows [r·⌈nA/W⌉, (r+1)·⌈nA/W⌉) of the
[nA, nB] matrix against all of B (B is replicated, 20 MB for config 4).  The result
is identical bit for bit for any world size (δ only selects values).  Two ways to
put the full matrix on every rank:

  * distribution="allgather": each rank writes its block locally, then one
    ``all_gather_into_tensor`` over NCCL (NVLink 5 / NVSwitch) assembles the
    matrix (blocks padded to equal height so that a single call suffices).
  * distribution="p2p" (fused): the matrix lives in torch symmetric memory; every
    rank's kernel (ffd_cdist_to) stores each finished result straight into ALL
    ranks' matrices through NVLink peer pointers while it computes, so the
    transfer overlaps the DP tile by tile and no collective moves the matrix.
    One device-side barrier (the symmetric-memory handle's) after the kernel
    publishes the writes.
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


def out_dtype(A):
    """Result dtype of the C ABI: int64 (exact) for int32 coordinates, else float32."""
    import torch
    return torch.int64 if A.dtype == torch.int32 else torch.float32


def assemble(block, n_rows: int, group=None):
    """All-gather equal-height row blocks [blk, nB] of every rank into [n_rows, nB]."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    blk, nB = block.shape
    full = torch.empty((world * blk, nB), dtype=block.dtype, device=block.device)
    dist.all_gather_into_tensor(full, block.contiguous(), group=group)
    return full[:n_rows]


def _check_distribution(distribution: str):
    if distribution not in ("allgather", "p2p"):
        raise ValueError(f"distribution must be 'allgather' or 'p2p', got {distribution!r}")


_SYMM_CACHE: dict = {}


def symmetric_matrix(shape, dtype, device, group=None):
    """A matrix in torch symmetric memory (every rank's copy mapped into every
    rank's address space over NVLink).  Returns (tensor, handle, peer pointers in
    rank order).  Cached per (shape, dtype, device, group): the rendezvous is a
    host-side exchange, done once; the next p2p call of the same shape reuses
    (and overwrites) the buffer."""
    import torch.distributed as dist
    import torch.distributed._symmetric_memory as symm_mem

    pg = group if group is not None else dist.group.WORLD
    key = (tuple(shape), dtype, str(device), id(pg))
    hit = _SYMM_CACHE.get(key)
    if hit is not None:
        return hit
    t = symm_mem.empty(*shape, dtype=dtype, device=device)
    hdl = symm_mem.rendezvous(t, pg)
    ptrs = [int(hdl.buffer_ptrs[r]) for r in range(hdl.world_size)]
    _SYMM_CACHE[key] = (t, hdl, ptrs)
    return t, hdl, ptrs


def cdist(A, B, norm: str = "l2", group=None, return_block: bool = False, distribution: str = "p2p"):
    """All-pairs δ_dF over the ranks of `group` (or the single local GPU).

    A [nA, lenA, dim], B [nB, lenB, dim] CUDA tensors, identical on every rank.
    Returns the full [nA, nB] matrix on every rank (float32, int64 for int32
    input), or only this rank's block with return_block=True (no distribution).
    distribution="p2p" returns the cached symmetric-memory matrix of this shape
    (see symmetric_matrix): the next p2p call of the same shape overwrites it, so
    clone it to keep it."""
    import torch.distributed as dist

    import paper_2404_05708_b200 as ffd

    _check_distribution(distribution)
    nA, nB = A.shape[0], B.shape[0]
    if group is None and not (dist.is_available() and dist.is_initialized()):
        return ffd.cdist(A, B, norm=norm)
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    r0, r1, blk = row_range(nA, world, rank)
    if return_block or distribution == "allgather":
        import torch
        block = torch.empty((blk, nB), dtype=out_dtype(A), device=A.device)
        if r1 > r0:
            ffd.cdist(A, B, norm=norm, rows=(r0, r1), out=block)
        if return_block:
            return block[: r1 - r0], (r0, r1)
        return assemble(block, nA, group)
    full, hdl, ptrs = symmetric_matrix((nA, nB), out_dtype(A), A.device, group)
    hdl.barrier()  # every rank's matrix is allocated before any peer writes into it
    if r1 > r0:
        ffd.cdist_to(A, B, ptrs, nB, norm=norm, rows=(r0, r1))
    hdl.barrier()  # device-side: every rank's kernel (and its peer stores) is done
    return full


# ---------------------------------------------------------------------------
# Self all-pairs matrix on W GPUs.  δ is symmetric,
# so only the upper triangle b ≥ a is evaluated.  Rank r owns the rows [r0, r1)
# and computes their columns [r0, n): its diagonal block as a self block (each
# unordered pair once) and the block right of it as a plain block.  Row
# boundaries balance the upper-triangle work Σ_a (n − a) across ranks.  The lower
# triangle is the transpose of the upper one (selection only: bit-identical to
# the single-GPU matrix): written as mirrored stores (p2p), or rebuilt from the
# gathered upper-triangle rows (allgather, blocks padded to one height H).
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


def upper_from_gathered(full, n: int, ranges):
    """The [n, n] matrix from gathered padded row blocks [W·H, n] that hold the
    upper-triangle rows of every rank (columns < r0 ignored): its upper triangle,
    mirrored."""
    import torch

    H = full.shape[0] // len(ranges)
    rows = torch.cat([torch.arange(r * H, r * H + (r1 - r0), device=full.device)
                      for r, (r0, r1) in enumerate(ranges)])
    upper = torch.triu(full[rows])
    return upper + torch.triu(upper, diagonal=1).T


def assemble_upper(block, n: int, ranges, group=None):
    """All-gather padded row blocks [H, n] holding the upper-triangle rows of every
    rank and mirror them into the full [n, n] matrix."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    H, _ = block.shape
    full = torch.empty((world * H, n), dtype=block.dtype, device=block.device)
    dist.all_gather_into_tensor(full, block.contiguous(), group=group)
    return upper_from_gathered(full, n, ranges)


def self_block(A, r0: int, r1: int, norm: str = "l2"):
    """Rank-local upper-triangle rows [r0, r1) of the self matrix, as an [r1 − r0, n]
    block (columns < r0 zero): the diagonal block by ffd_cdist_self, the block to
    its right by ffd_cdist."""
    import torch

    import paper_2404_05708_b200 as ffd

    n = A.shape[0]
    block = torch.zeros((r1 - r0, n), dtype=out_dtype(A), device=A.device)
    if r1 > r0:
        block[:, r0:r1] = ffd.cdist_self(A[r0:r1].contiguous(), norm=norm)
        if r1 < n:
            block[:, r1:] = ffd.cdist(A[r0:r1].contiguous(), A[r1:].contiguous(), norm=norm)
    return block


def cdist_self(A, norm: str = "l2", group=None, distribution: str = "p2p"):
    """All-pairs δ_dF of the set A against itself over the ranks of `group` (or the
    single local GPU): about half the work of cdist(A, A)."""
    import torch
    import torch.distributed as dist

    import paper_2404_05708_b200 as ffd

    _check_distribution(distribution)
    n = A.shape[0]
    if group is None and not (dist.is_available() and dist.is_initialized()):
        return ffd.cdist_self(A, norm=norm)
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    ranges = self_row_ranges(n, world)
    r0, r1 = ranges[rank]
    if distribution == "allgather":
        H = max(1, max(b - a for a, b in ranges))
        block = torch.zeros((H, n), dtype=out_dtype(A), device=A.device)
        block[: r1 - r0] = self_block(A, r0, r1, norm)
        return assemble_upper(block, n, ranges, group)
    full, hdl, ptrs = symmetric_matrix((n, n), out_dtype(A), A.device, group)
    hdl.barrier()
    A = A.contiguous()
    if r1 > r0:
        # diagonal block: each unordered pair inside the shard once, both places
        ffd.cdist_to(A, A[r0:r1], ptrs, n, norm=norm, rows=(r0, r1), self_mode=True, col_offset=r0)
        if r1 < n:  # right of it: (a, b) and its mirror (b, a)
            ffd.cdist_to(A, A[r1:], ptrs, n, norm=norm, rows=(r0, r1), col_offset=r1, mirror=True)
    hdl.barrier()
    return full


# ---------------------------------------------------------------------------
# One very long pair over W GPUs.  The long-pair wavefront is a
# chain of row bands (linear memory); the chain simply continues
# across GPUs.  Rank r computes a contiguous range of rows of the rows curve (the
# shorter one) with ffd_long_pair_shard; its last band stores its bottom row,
# slot by slot, straight into the next rank's ring in symmetric memory (NVLink
# peer stores), where that rank's first band polls it.  A ring holds a whole
# stream, so no rank ever waits for its consumer; the result is written by the
# rank that holds the last row and broadcast.  Bit-identical to one GPU (the DP
# only selects values; the bands and their inputs are the same).
# ---------------------------------------------------------------------------
def long_pair_row_ranges(rows: int, world: int, align: int) -> list[tuple[int, int]]:
    """Contiguous row ranges [r0, r1) covering [0, rows), boundaries at multiples of
    `align`, balanced; ranks beyond ⌈rows / align⌉ get an empty range at the end."""
    if world < 1 or rows < 1 or align < 1:
        raise ValueError("bad long_pair_row_ranges arguments")
    active = min(world, -(-rows // align))
    bounds = [min(rows, round(r * rows / active / align) * align) for r in range(active)] + [rows]
    ranges = [(bounds[r], bounds[r + 1]) for r in range(active)]
    return ranges + [(rows, rows)] * (world - active)


_LONG_RINGS: dict = {}


def long_pair(p, q, norm: str = "l2", group=None):
    """δ_dF of ONE pair (p [n, dim], q [m, dim] fp32 CUDA tensors, identical on every
    rank) with its rows split over the ranks of `group`.  Returns float32[1] on
    every rank."""
    import torch
    import torch.distributed as dist
    import torch.distributed._symmetric_memory as symm_mem

    import paper_2404_05708_b200 as ffd

    n, m = p.shape[0], q.shape[0]
    if group is None and not (dist.is_available() and dist.is_initialized()):
        off = torch.zeros(2, dtype=torch.int64, device=p.device)
        lens = torch.tensor([n, m], dtype=torch.int32, device=p.device)
        return ffd.batch(p, q, off, lens, norm=norm)
    pg = group if group is not None else dist.group.WORLD
    world, rank = dist.get_world_size(pg), dist.get_rank(pg)
    rows = min(n, m)
    ranges = long_pair_row_ranges(rows, world, ffd.long_pair_row_align())
    nbytes = ffd.long_pair_ring_bytes(n, m)
    key = (nbytes, str(p.device), id(pg))
    ent = _LONG_RINGS.get(key)
    if ent is None:
        ring = symm_mem.empty(nbytes, dtype=torch.uint8, device=p.device)
        ring.zero_()
        hdl = symm_mem.rendezvous(ring, pg)
        ent = _LONG_RINGS[key] = {"ring": ring, "hdl": hdl, "tag": 0,
                                  "ptrs": [int(hdl.buffer_ptrs[r]) for r in range(world)]}
    slots = nbytes // 8
    if ent["tag"] + 2 * slots >= 2 ** 32:  # tags are 32-bit: start over on zeroed rings
        ent["hdl"].barrier()
        ent["ring"].zero_()
        ent["tag"] = 0
    tag = ent["tag"]
    ent["tag"] += slots
    out = torch.full((1,), float("nan"), dtype=torch.float32, device=p.device)
    ent["hdl"].barrier()  # every rank is done reading its ring from the previous call
    r0, r1 = ranges[rank]
    if r1 > r0:
        nxt = (ent["ptrs"][rank + 1], nbytes) if r1 < rows else None
        ffd.long_pair_shard(p, q, (r0, r1), norm, in_ring=ent["ring"] if r0 > 0 else None, in_tag=tag,
                            out_ring=nxt, out_tag=tag, out=out)
    last = max(r for r in range(world) if ranges[r][1] == rows and ranges[r][1] > ranges[r][0])
    dist.broadcast(out, src=dist.get_global_rank(pg, last) if group is not None else last, group=group)
    return out
