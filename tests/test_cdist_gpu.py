"""Parity of ffd_cdist (CUDA, through the C ABI) against the CPU oracle."""
import numpy as np
import pytest

import oracle
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


def check(got, A, B, ia, ib, norm):
    ref = oracle.cdist_entries(A, B, ia, ib, norm)
    mir = oracle.cdist_entries(A, B, ia, ib, norm, mirror=True)
    err = np.abs(got.astype(np.float64) - ref)
    assert (err <= 1e-5 * np.abs(ref)).all(), f"max rel err {(err / np.maximum(np.abs(ref), 1e-30)).max()}"
    assert np.array_equal(got, mir), f"{(got != mir).sum()} entries differ from the fp32 mirror"


@pytest.mark.parametrize("lenA,lenB,norm,dim", [(128, 128, "l2", 2), (37, 90, "l2", 2), (128, 200, "l1", 2),
                                                (250, 64, "linf", 2), (500, 33, "sql2", 2), (1, 5, "l2", 2),
                                                (64, 1, "l2", 2), (100, 120, "l2", 3)])
def test_small_full_matrix(ffd, lenA, lenB, norm, dim):
    cfg = workload.CONFIGS[4].scaled(nA=23, nB=301, length=lenA, dim=dim)
    A = workload.gen_set(cfg, "A")
    B = workload.gen_set(cfg.scaled(length=lenB), "B")
    got = ffd.cdist(torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda(), norm=norm).cpu().numpy()
    ia = np.repeat(np.arange(23), 301)
    ib = np.tile(np.arange(301), 23)
    check(got.ravel(), A, B, ia, ib, norm)


def test_shard_rows_and_ld(ffd):
    cfg = workload.CONFIGS[4].scaled(nA=50, nB=140, length=128)
    A = torch.from_numpy(workload.gen_set(cfg, "A")).cuda()
    B = torch.from_numpy(workload.gen_set(cfg, "B")).cuda()
    full = ffd.cdist(A, B, "l2")
    out = torch.full((20, 150), -1.0, device="cuda")
    ffd.cdist(A, B, "l2", rows=(13, 33), out=out, ld_out=150)
    assert torch.equal(out[:, :140], full[13:33])
    assert (out[:, 140:] == -1).all()          # nothing written past nB


def test_config4_full_size_sampled(ffd):
    """Full BASELINE config 4 (20k × 20k, L=128) in the bench launch shape;
    sampled entries + one full row and column checked against the oracle."""
    cfg = workload.CONFIGS[4]
    A = workload.gen_set(cfg, "A")
    B = workload.gen_set(cfg, "B")
    got = ffd.cdist(torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda(), "l2")
    n = 3000
    ia = workload.sample_indices(cfg, 0, n, cfg.nA)
    ib = workload.sample_indices(cfg, 1, n, cfg.nB)
    ia = np.concatenate([ia, np.full(400, 12345), np.arange(400) * 50])
    ib = np.concatenate([ib, np.arange(400) * 50, np.full(400, 777)])
    sel = got[torch.from_numpy(ia).cuda(), torch.from_numpy(ib).cuda()].cpu().numpy()
    check(sel, A, B, ia, ib, "l2")
    # properties at full size: finite, non-negative, diagonal-free sanity
    assert torch.isfinite(got).all() and (got >= 0).all()


def test_cdist_self_matches_full_and_oracle(ffd):
    """ffd_cdist_self (each unordered pair evaluated once, mirrored) equals
    ffd_cdist(A, A) bit for bit — δ is symmetric exactly in fp32 — on the full
    range and on shards, with oracle spot checks."""
    cfg = workload.CONFIGS[4].scaled(nA=300, nB=300, length=70)
    A_h = workload.gen_set(cfg, "A")
    A = torch.from_numpy(A_h).cuda()
    full = ffd.cdist(A, A, "l2")
    selfm = ffd.cdist_self(A, "l2")
    assert torch.equal(full, selfm)
    assert torch.equal(selfm, selfm.T)
    assert (torch.diagonal(selfm) == 0).all()
    for r0, r1 in [(0, 1), (37, 180), (250, 300)]:
        blk = ffd.cdist_self(A, "l2", rows=(r0, r1))
        assert torch.equal(blk, full[r0:r1])
    ia = np.array([0, 5, 299, 123, 77], np.int64)
    ib = np.array([299, 5, 0, 200, 76], np.int64)
    check(selfm[torch.from_numpy(ia).cuda(), torch.from_numpy(ib).cuda()].cpu().numpy(), A_h, A_h, ia, ib, "l2")


def _dense_pairs(A, B, r0, r1):
    """oracle batch layout of all (a, b), a ∈ [r0, r1), over the flattened sets"""
    nA, LA, dim = A.shape
    nB, LB, _ = B.shape
    a = np.repeat(np.arange(r0, r1), nB)
    b = np.tile(np.arange(nB), r1 - r0)
    off = np.concatenate([a * LA, b * LB]).astype(np.int64)
    lens = np.concatenate([np.full(len(a), LA), np.full(len(b), LB)]).astype(np.int32)
    return A.reshape(-1, dim), B.reshape(-1, dim), off, lens


@pytest.mark.parametrize("dim,dtype,lenA,lenB,norm", [
    (1, "f", 40, 50, "l2"), (4, "f", 30, 33, "l1"), (2, "f", 700, 90, "l2"),
    (2, "i", 60, 70, "sql2"), (3, "i", 45, 20, "linf")])
def test_cdist_general_shapes(ffd, dim, dtype, lenA, lenB, norm):
    """shapes outside the dedicated all-pairs kernel (int32, dim 1/4, A-curves
    longer than 512 points) go through the batch kernels: same results"""
    rng = np.random.default_rng(dim * 100 + lenA)
    nA, nB = 9, 7
    if dtype == "i":
        A = np.cumsum(rng.integers(-8, 9, size=(nA, lenA, dim)), 1).astype(np.int32)
        B = np.cumsum(rng.integers(-8, 9, size=(nB, lenB, dim)), 1).astype(np.int32)
    else:
        A = np.cumsum(rng.normal(size=(nA, lenA, dim)), 1).astype(np.float32)
        B = np.cumsum(rng.normal(size=(nB, lenB, dim)), 1).astype(np.float32)
    got = ffd.cdist(torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda(), norm, rows=(2, 8)).cpu().numpy()
    p, q, off, lens = _dense_pairs(A, B, 2, 8)
    if dtype == "i":
        ref = oracle.batch(p, q, off, lens, dim, norm).reshape(6, nB)
        assert np.array_equal(got, ref)
    else:
        mir = oracle.batch(p, q, off, lens, dim, norm, mirror=True).reshape(6, nB)
        assert np.array_equal(got, mir)


def test_cdist_self_general_shape(ffd):
    rng = np.random.default_rng(8)
    A = np.cumsum(rng.normal(size=(11, 600, 2)), 1).astype(np.float32)   # > 512 points
    got = ffd.cdist_self(torch.from_numpy(A).cuda(), "l2").cpu().numpy()
    p, q, off, lens = _dense_pairs(A, A, 0, 11)
    assert np.array_equal(got, oracle.batch(p, q, off, lens, 2, "l2", mirror=True).reshape(11, 11))
