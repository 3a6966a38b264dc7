"""Parity of ffd_dist_sum (Σ_ij d_ij, the paper's "upper limit" baseline,
PAPER L300, L304–L305, through the C ABI) against the fp64 CPU oracle, within
the bound include/ffd.h states: (35 + 2·dim)·2⁻²⁴ relative (fp32 column sums
of ≤ 32 positive terms, approximate square root)."""
import numpy as np
import pytest

import oracle

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ffd():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2404_05708_b200 as ffd
    ffd.lib()
    return ffd


def make(rng, lens, dim=2, one_vs_many=False):
    B = len(lens) // 2
    lens = np.asarray(lens, np.int32)
    if one_vs_many:
        lens[B:] = lens[B]
    off = np.zeros(2 * B, np.int64)
    off[1:B] = np.cumsum(lens[:B - 1])
    if not one_vs_many:
        off[B + 1:] = np.cumsum(lens[B:-1])
    nq = int(lens[B]) if one_vs_many else int(lens[B:].sum())
    p = np.cumsum(rng.normal(size=(int(lens[:B].sum()), dim)), 0).astype(np.float32)
    q = np.cumsum(rng.normal(size=(nq, dim)), 0).astype(np.float32)
    return p, q, off, lens


def run(ffd, p, q, off, lens, norm):
    args = [torch.from_numpy(a).cuda() for a in (p, q, off, lens)]
    return ffd.dist_sum(*args, norm=norm).cpu().numpy()


def check(got, p, q, off, lens, dim, norm):
    ref = oracle.dist_sum_batch(p, q, off, lens, dim, norm)
    tol = (35 + 2 * dim) * 2.0 ** -24
    bad = np.abs(got - ref) > tol * np.abs(ref) + 1e-30
    assert not bad.any(), (norm, dim, np.flatnonzero(bad)[:5], got[bad][:5], ref[bad][:5])


@pytest.mark.parametrize("dim", [1, 2, 3, 4])
@pytest.mark.parametrize("norm", ["l1", "l2", "linf", "sql2"])
def test_dist_sum_ragged(ffd, dim, norm):
    """ragged lengths from 1 to several 32×256 tiles, with ragged tails"""
    rng = np.random.default_rng(100 + dim)
    B = 40
    lens = rng.integers(1, 700, size=2 * B)
    lens[:4] = [1, 1, 33, 257]
    lens[B:B + 4] = [1, 300, 1, 513]
    p, q, off, lens = make(rng, lens, dim)
    check(run(ffd, p, q, off, lens, norm), p, q, off, lens, dim, norm)


def test_dist_sum_one_vs_many_and_determinism(ffd):
    """the paper's setting (N curves against one q, every q offset 0);
    small B spreads one pair over many CTAs (splits), results bit-stable"""
    rng = np.random.default_rng(7)
    for B in (1, 3, 64):
        p, q, off, lens = make(rng, rng.integers(200, 1500, size=2 * B), 2, one_vs_many=True)
        a = run(ffd, p, q, off, lens, "l2")
        check(a, p, q, off, lens, 2, "l2")
        assert np.array_equal(a, run(ffd, p, q, off, lens, "l2"))


def test_dist_sum_e1_shape_sampled(ffd):
    """E1's largest point (N = 2^14 walks of 2^10 points vs one q):
    the oracle on 16 sampled pairs"""
    import workload
    cfg = workload.CONFIGS[101].scaled(pairs=4096, len_p=(1024, 1024), len_q=(1024, 1024))
    b = workload.gen_batch(cfg)
    N = 4096
    q = b.q[:1024].copy()
    off = np.concatenate([b.offsets[:N], np.zeros(N, np.int64)])
    got = run(ffd, b.p, q, off, b.lengths, "l2")
    sel = np.random.default_rng(0).choice(N, 16, replace=False)
    offs = np.concatenate([off[sel], off[N + sel]])
    ln = np.concatenate([b.lengths[sel], b.lengths[N + sel]])
    ref = oracle.dist_sum_batch(b.p, q, offs, ln, 2, "l2")
    assert np.all(np.abs(got[sel] - ref) <= 39 * 2.0 ** -24 * ref)


def test_dist_sum_edges(ffd):
    rng = np.random.default_rng(3)
    p, q, off, lens = make(rng, [5, 0, 7, 4], 2)
    got = run(ffd, p, q, off, lens, "l2")
    assert np.isnan(got[1]) and np.isfinite(got[0])
    pi = torch.zeros((4, 2), dtype=torch.int32, device="cuda")
    o = torch.zeros(2, dtype=torch.int64, device="cuda")
    ln = torch.ones(2, dtype=torch.int32, device="cuda")
    with pytest.raises(ffd.FFDError):
        ffd.dist_sum(pi, pi, o, ln, norm="sql2")
    empty = ffd.dist_sum(torch.zeros((1, 2), device="cuda"), torch.zeros((1, 2), device="cuda"),
                         torch.zeros(0, dtype=torch.int64, device="cuda"),
                         torch.zeros(0, dtype=torch.int32, device="cuda"))
    assert empty.numel() == 0
