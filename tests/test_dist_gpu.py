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


@pytest.mark.parametrize("W", [2, 3, 8])
def test_long_pair_shards_emulated(ffd, W):
    """ffd_long_pair_shard over W emulated GPUs, run one after another on this GPU
    (the rings hold a whole stream, so no range waits for its consumer): the band
    chain crosses the ranges through the rings and the result is bit-identical to
    the single-call long-pair kernel, for two calls with the tag base advanced
    (no re-zeroing) and with the ranges forced into several passes (1 CTA)."""
    from paper_2404_05708_b200.dist import long_pair_row_ranges
    rng = np.random.default_rng(40 + W)
    n, m = 20000, 21001
    p = torch.from_numpy(np.cumsum(rng.normal(size=(n, 2)), 0).astype(np.float32)).cuda()
    q = torch.from_numpy(np.cumsum(rng.normal(size=(m, 2)), 0).astype(np.float32)).cuda()
    off = torch.zeros(2, dtype=torch.int64, device="cuda")
    lens = torch.tensor([n, m], dtype=torch.int32, device="cuda")
    nbytes = ffd.long_pair_ring_bytes(n, m)
    rings = [torch.zeros(nbytes, dtype=torch.uint8, device="cuda") for _ in range(W)]
    ranges = long_pair_row_ranges(min(n, m), W, ffd.long_pair_row_align())
    for norm in ("l2", "linf"):
        full = ffd.batch(p, q, off, lens, norm=norm).item()
        for call, ctas in enumerate(("", "", "1")):
            if ctas:
                os.environ["FFD_LONG_CTAS"] = ctas
            try:
                tag = (call + (norm == "linf") * 3) * (nbytes // 8)
                out = torch.full((1,), float("nan"), device="cuda")
                for r, (r0, r1) in enumerate(ranges):
                    if r1 == r0:
                        continue
                    nxt = (rings[r + 1].data_ptr(), nbytes) if r1 < min(n, m) else None
                    ffd.long_pair_shard(p, q, (r0, r1), norm, in_ring=rings[r] if r0 > 0 else None, in_tag=tag,
                                        out_ring=nxt, out_tag=tag, out=out)
            finally:
                os.environ.pop("FFD_LONG_CTAS", None)
            assert out.item() == full, (W, norm, call, out.item(), full)


def test_long_pair_over_nccl(ffd, nccl_group):
    """dist.long_pair through a real process group (world size 1: one range) and
    its symmetric-memory ring, against the single-GPU call."""
    from paper_2404_05708_b200 import dist as fdist
    rng = np.random.default_rng(44)
    p = torch.from_numpy(np.cumsum(rng.normal(size=(5000, 2)), 0).astype(np.float32)).cuda()
    q = torch.from_numpy(np.cumsum(rng.normal(size=(7000, 2)), 0).astype(np.float32)).cuda()
    off = torch.zeros(2, dtype=torch.int64, device="cuda")
    lens = torch.tensor([5000, 7000], dtype=torch.int32, device="cuda")
    for _ in range(2):
        got = fdist.long_pair(p, q, "l1").item()
        assert got == ffd.batch(p, q, off, lens, norm="l1").item()


def test_long_pair_shard_rejects_bad_ranges(ffd):
    p = torch.zeros((2000, 2), device="cuda")
    q = torch.zeros((3000, 2), device="cuda")
    ring = torch.zeros(ffd.long_pair_ring_bytes(2000, 3000), dtype=torch.uint8, device="cuda")
    with pytest.raises(ffd.FFDError):
        ffd.long_pair_shard(p, q, (100, 2000), in_ring=ring)              # unaligned begin
    with pytest.raises(ffd.FFDError):
        ffd.long_pair_shard(p, q, (0, 1000))                              # no out ring
    with pytest.raises(ffd.FFDError):
        ffd.long_pair_shard(p, q, (512, 2000))                            # no in ring
