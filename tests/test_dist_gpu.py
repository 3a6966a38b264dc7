"""The multi-GPU product path on the one GPU a test box has:

  * row shards for W = 2, 4, 8 computed by ffd_cdist / the self-block split and
    concatenated are bit-identical to the W = 1 matrix (δ only selects values);
  * the fused distribution (ffd_cdist_to) with W destination matrices: every
    "rank" r of an emulated W-rank job writes its shard into ALL W matrices (on
    a multi-GPU node those are NVLink peer mappings of the other GPUs' matrices;
    here W buffers of this GPU stand in for them — the ranks' kernels do not
    wait on one another, so running them one after the other is exact);
  * dist.cdist / dist.cdist_self through a real NCCL process group (world size
    1), with both distributions (all-gather and symmetric-memory P2P).
"""
import os
import socket

import numpy as np
import pytest

import workload

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ffd():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2404_05708_b200 as ffd
    ffd.lib()
    return ffd


def sets(kind, nA=301, nB=257, L=128, dim=2):
    if kind == "f32":
        cfg = workload.CONFIGS[4].scaled(nA=nA, nB=nB, length=L, dim=dim)
        return (torch.from_numpy(workload.gen_set(cfg, "A")).cuda(),
                torch.from_numpy(workload.gen_set(cfg, "B")).cuda(), "l2")
    rng = np.random.default_rng(5)
    A = np.cumsum(rng.integers(-8, 9, size=(nA, L, dim)), 1).astype(np.int32)
    B = np.cumsum(rng.integers(-8, 9, size=(nB, L, dim)), 1).astype(np.int32)
    return torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda(), "sql2"


@pytest.mark.parametrize("kind", ["f32", "i32"])
def test_row_shards_bit_identical(ffd, kind):
    from paper_2404_05708_b200.dist import row_range, self_block, self_row_ranges, upper_from_gathered
    A, B, norm = sets(kind)
    full = ffd.cdist(A, B, norm=norm)
    full_self = ffd.cdist_self(A, norm=norm)
    n = A.shape[0]
    for W in (2, 4, 8):
        blocks = [ffd.cdist(A, B, norm=norm, rows=row_range(A.shape[0], W, r)[:2]) for r in range(W)]
        assert torch.equal(torch.cat(blocks), full), W
        ranges = self_row_ranges(n, W)
        H = max(r1 - r0 for r0, r1 in ranges)
        gathered = torch.zeros((W * H, n), dtype=full_self.dtype, device="cuda")
        for r, (r0, r1) in enumerate(ranges):
            gathered[r * H: r * H + r1 - r0] = self_block(A, r0, r1, norm)
        assert torch.equal(upper_from_gathered(gathered, n, ranges), full_self), W


@pytest.mark.parametrize("kind", ["f32", "i32"])
@pytest.mark.parametrize("W", [1, 3, 8])
def test_fused_distribution_emulated_ranks(ffd, kind, W):
    """ffd_cdist_to: each emulated rank stores its shard into all W matrices."""
    from paper_2404_05708_b200.dist import out_dtype, row_range, self_row_ranges
    A, B, norm = sets(kind)
    nA, nB = A.shape[0], B.shape[0]
    full = ffd.cdist(A, B, norm=norm)
    mats = [torch.full((nA, nB), -1, dtype=out_dtype(A), device="cuda") for _ in range(W)]
    ptrs = [m.data_ptr() for m in mats]
    for r in range(W):
        r0, r1, _ = row_range(nA, W, r)
        if r1 > r0:
            ffd.cdist_to(A, B, ptrs, nB, norm=norm, rows=(r0, r1))
    for m in mats:
        assert torch.equal(m, full)
    # the self matrix: diagonal self blocks + mirrored blocks to their right
    full_self = ffd.cdist_self(A, norm=norm)
    mats = [torch.full((nA, nA), -1, dtype=out_dtype(A), device="cuda") for _ in range(W)]
    ptrs = [m.data_ptr() for m in mats]
    for r0, r1 in self_row_ranges(nA, W):
        if r1 > r0:
            ffd.cdist_to(A, A[r0:r1], ptrs, nA, norm=norm, rows=(r0, r1), self_mode=True, col_offset=r0)
            if r1 < nA:
                ffd.cdist_to(A, A[r1:], ptrs, nA, norm=norm, rows=(r0, r1), col_offset=r1, mirror=True)
    for m in mats:
        assert torch.equal(m, full_self)


def test_cdist_to_rejects_bad_args(ffd):
    A, B, norm = sets("f32", nA=4, nB=3, L=8)
    m = torch.zeros((4, 3), device="cuda")
    with pytest.raises(ffd.FFDError):
        ffd.cdist_to(A, B, [m.data_ptr()] * 9, 3, norm=norm)           # > 8 destinations
    with pytest.raises(ffd.FFDError):
        ffd.cdist_to(A, B, [m.data_ptr()], 2, norm=norm)               # ld_out < nB
    with pytest.raises(ffd.FFDError):
        ffd.cdist_to(A, A, [m.data_ptr()], 4, norm=norm, self_mode=True, mirror=True)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.fixture(scope="module")
def nccl_group():
    import torch.distributed as dist
    if dist.is_initialized():
        yield dist.group.WORLD
        return
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{_free_port()}", rank=0, world_size=1,
                            device_id=torch.device("cuda", 0))
    yield dist.group.WORLD
    dist.destroy_process_group()


@pytest.mark.parametrize("distribution", ["allgather", "p2p"])
@pytest.mark.parametrize("kind", ["f32", "i32"])
def test_dist_product_over_nccl(ffd, nccl_group, distribution, kind):
    from paper_2404_05708_b200 import dist as fdist
    A, B, norm = sets(kind, nA=211, nB=173)
    full = fdist.cdist(A, B, norm=norm, distribution=distribution)
    assert full.dtype == (torch.int64 if kind == "i32" else torch.float32)
    assert torch.equal(full, ffd.cdist(A, B, norm=norm))
    selfm = fdist.cdist_self(A, norm=norm, distribution=distribution)
    assert torch.equal(selfm, ffd.cdist_self(A, norm=norm))
    blk, rows = fdist.cdist(A, B, norm=norm, return_block=True)
    assert rows == (0, A.shape[0]) and torch.equal(blk, full)
