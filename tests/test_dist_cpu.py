"""Multi-rank sharding + all-gather logic of paper_2404_05708_b200.dist on CPU
(gloo, world size 2 and 3).  The per-rank block is computed by the oracle here
(test side) — the product path computes it with ffd_cdist on the GPU."""
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
