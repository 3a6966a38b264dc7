"""Multi-rank sharding + all-gather logic of paper_2404_05708_b200.dist on CPU
(gloo, world size 2 and 3).  The per-rank block is computed by the oracle here
(test side) — the product path computes it with ffd_cdist on the GPU.  The
product functions dist.cdist / dist.cdist_self themselves run here with the
library's block calls (ffd.cdist, ffd.cdist_self) replaced by oracle stand-ins,
which is the only way to run them without a GPU; tests/test_dist_gpu.py runs
them for real through NCCL."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2404_05708_b200.dist import assemble, assemble_upper, row_range, self_row_ranges


def test_row_range_covers_exactly():
    for n in (1, 7, 20000, 20001):
        for w in (1, 2, 3, 4, 8):
            rows = []
            for r in range(w):
                r0, r1, blk = row_range(n, w, r)
                assert r1 - r0 <= blk
                rows.extend(range(r0, r1))
            assert rows == list(range(n))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import oracle
    import workload
    cfg = workload.CONFIGS[4].scaled(nA=11, nB=7, length=16)
    A, B = workload.gen_set(cfg, "A"), workload.gen_set(cfg, "B")
    r0, r1, blk = row_range(cfg.nA, world, rank)
    block = torch.zeros((blk, cfg.nB), dtype=torch.float32)
    if r1 > r0:
        ia = np.repeat(np.arange(r0, r1), cfg.nB)
        ib = np.tile(np.arange(cfg.nB), r1 - r0)
        block[: r1 - r0] = torch.from_numpy(
            oracle.cdist_entries(A, B, ia, ib, "l2", mirror=True).reshape(r1 - r0, cfg.nB))
    full = assemble(block, cfg.nA)
    if rank == 0:
        ia = np.repeat(np.arange(cfg.nA), cfg.nB)
        ib = np.tile(np.arange(cfg.nB), cfg.nA)
        ref = oracle.cdist_entries(A, B, ia, ib, "l2", mirror=True).reshape(cfg.nA, cfg.nB)
        q.put(bool(np.array_equal(full.numpy(), ref)))
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_gloo_assemble(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    assert q.get(timeout=10) is True


def test_self_row_ranges_balanced():
    for n in (1, 5, 100, 20000):
        for w in (1, 2, 3, 8):
            rs = self_row_ranges(n, w)
            assert rs[0][0] == 0 and rs[-1][1] == n
            assert all(rs[i][1] == rs[i + 1][0] for i in range(w - 1))
            work = [sum(n - a for a in range(r0, r1)) for r0, r1 in rs]
            if n >= 100:
                assert max(work) - min(work) <= 2 * n   # within two rows of the ideal split


def _worker_self(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import oracle
    import workload
    cfg = workload.CONFIGS[4].scaled(nA=13, length=12)
    A = workload.gen_set(cfg, "A")
    n = cfg.nA
    ranges = self_row_ranges(n, world)
    H = max(r1 - r0 for r0, r1 in ranges)
    r0, r1 = ranges[rank]
    block = torch.zeros((H, n), dtype=torch.float32)
    if r1 > r0:   # this rank's upper-triangle rows, computed test-side by the oracle
        ia = np.repeat(np.arange(r0, r1), n - r0)
        ib = np.tile(np.arange(r0, n), r1 - r0)
        block[: r1 - r0, r0:] = torch.from_numpy(
            oracle.cdist_entries(A, A, ia, ib, "l2", mirror=True).reshape(r1 - r0, n - r0))
    full = assemble_upper(block, n, ranges)
    if rank == 0:
        ia = np.repeat(np.arange(n), n)
        ib = np.tile(np.arange(n), n)
        ref = oracle.cdist_entries(A, A, ia, ib, "l2", mirror=True).reshape(n, n)
        q.put(bool(np.array_equal(full.numpy(), ref)))
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_gloo_assemble_self(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker_self, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    assert q.get(timeout=10) is True


def _oracle_standins():
    """ffd.cdist / ffd.cdist_self stand-ins computed by the oracle on CPU tensors
    (float32 -> fp32 mirror, int32 -> exact int64), same signatures."""
    import oracle
    import paper_2404_05708_b200 as ffd

    def block(A, B, norm, r0, r1):
        A_, B_ = A.numpy(), B.numpy()
        nB = B_.shape[0]
        ia = np.repeat(np.arange(r0, r1), nB)
        ib = np.tile(np.arange(nB), r1 - r0)
        if A_.dtype == np.int32:
            out = np.array([oracle.pair(A_[a], B_[b], norm) for a, b in zip(ia, ib)], np.int64)
        else:
            out = oracle.cdist_entries(A_, B_, ia, ib, norm, mirror=True)
        return torch.from_numpy(out.reshape(r1 - r0, nB))

    def cdist(A, B, norm="l2", rows=None, out=None, **kw):
        r0, r1 = (0, A.shape[0]) if rows is None else rows
        blk = block(A, B, norm, r0, r1)
        if out is None:
            return blk
        out[: r1 - r0] = blk
        return out

    def cdist_self(A, norm="l2", rows=None, out=None, **kw):
        return cdist(A, A, norm=norm, rows=rows, out=out)

    ffd.cdist = cdist
    ffd.cdist_self = cdist_self
    return block


def _worker_product(rank, world, port, q, kind):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import workload
    from paper_2404_05708_b200 import dist as fdist
    block = _oracle_standins()
    cfg = workload.CONFIGS[4].scaled(nA=11, nB=7, length=14)
    if kind == "i32":
        cfg = cfg.scaled(dtype="i32", walk="int", norm="sql2")
        A = torch.from_numpy(np.cumsum(np.random.default_rng(1).integers(-9, 10, size=(11, 14, 2)), 1).astype(np.int32))
        B = torch.from_numpy(np.cumsum(np.random.default_rng(2).integers(-9, 10, size=(7, 14, 2)), 1).astype(np.int32))
        norm = "sql2"
    else:
        A = torch.from_numpy(workload.gen_set(cfg, "A"))
        B = torch.from_numpy(workload.gen_set(cfg, "B"))
        norm = "l2"
    full = fdist.cdist(A, B, norm=norm, distribution="allgather")
    selfm = fdist.cdist_self(A, norm=norm, distribution="allgather")
    blk, (r0, r1) = fdist.cdist(A, B, norm=norm, return_block=True)
    ok = True
    if rank == 0:
        ref = block(A, B, norm, 0, A.shape[0])
        ref_self = block(A, A, norm, 0, A.shape[0])
        ok = (torch.equal(full, ref) and torch.equal(selfm, ref_self) and full.dtype == ref.dtype
              and selfm.dtype == ref.dtype)
    ok = ok and torch.equal(blk, block(A, B, norm, r0, r1))
    q.put(bool(ok))
    dist.destroy_process_group()


@pytest.mark.parametrize("world,kind", [(2, "f32"), (3, "f32"), (2, "i32")])
def test_gloo_product_cdist(world, kind):
    """dist.cdist and dist.cdist_self themselves (allgather distribution) over gloo:
    sharding, padding, gather and the upper-triangle mirror, float and int32
    (int64 results; cdist_self cast int results to float32)."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker_product, args=(r, world, port, q, kind)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(180)
        assert p.exitcode == 0
    assert all(q.get(timeout=10) is True for _ in range(world))


def test_long_pair_row_ranges():
    from paper_2404_05708_b200.dist import long_pair_row_ranges
    for rows in (1, 511, 512, 513, 20000, 262144, 1250000):
        for w in (1, 2, 3, 4, 8):
            rs = long_pair_row_ranges(rows, w, 512)
            assert len(rs) == w and rs[0][0] == 0
            covered = [x for r0, r1 in rs for x in (r0, r1) if r1 > r0]
            assert all(rs[i][1] == rs[i + 1][0] for i in range(w - 1))
            assert rs[-1][1] == rows
            for r0, r1 in rs:
                assert r1 >= r0
                if r1 > r0:
                    assert r0 % 512 == 0 and (r1 == rows or r1 % 512 == 0)
            sizes = [r1 - r0 for r0, r1 in rs if r1 > r0]
            assert covered and max(sizes) - min(sizes) <= 1024 or len(sizes) == 1
