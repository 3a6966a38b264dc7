"""Parity of ffd_batch_dtw (DTW, PAPER Appendix B, through the C ABI)
against the CPU oracle: bit-exact against the fp32 mirror of the kernels'
operation order, and within the rounding bound of an (n+m)-term fp32 sum of the
fp64 oracle."""
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


def make(rng, lens, dim=2):
    B = len(lens) // 2
    lens = np.asarray(lens, np.int32)
    off = np.zeros(2 * B, np.int64)
    off[1:B] = np.cumsum(lens[:B - 1])
    off[B + 1:] = np.cumsum(lens[B:-1])
    p = np.cumsum(rng.normal(size=(int(lens[:B].sum()), dim)), 0).astype(np.float32)
    q = np.cumsum(rng.normal(size=(int(lens[B:].sum()), dim)), 0).astype(np.float32)
    return p, q, off, lens


def run(ffd, p, q, off, lens, norm):
    args = [torch.from_numpy(a).cuda() for a in (p, q, off, lens)]
    return ffd.dtw_batch(*args, norm=norm).cpu().numpy()


def check(got, p, q, off, lens, dim, norm):
    B = len(lens) // 2
    mir = oracle.dtw_batch(p, q, off, lens, dim, norm, mirror=True)
    ref = oracle.dtw_batch(p, q, off, lens, dim, norm)
    bad = got != mir
    assert not bad.any(), f"{bad.sum()} differ from the fp32 mirror; first {np.nonzero(bad)[0][:5]}"
    tol = (lens[:B].astype(np.float64) + lens[B:] + dim + 2) * 2.0 ** -24 * np.abs(ref)
    assert (np.abs(got - ref) <= tol).all()


@pytest.mark.parametrize("dim", [1, 2, 3, 4])
@pytest.mark.parametrize("norm", ["l2", "sql2", "l1", "linf"])
def test_dtw_random(ffd, norm, dim):
    rng = np.random.default_rng(300 + dim * 11 + len(norm))
    lens = rng.integers(1, 700, size=2 * 120)
    p, q, off, lens = make(rng, lens, dim)
    check(run(ffd, p, q, off, lens, norm), p, q, off, lens, dim, norm)


def test_dtw_edges_and_bands(ffd):
    """lengths around lane/band boundaries, multi-band rows, n ≫ m and m ≫ n"""
    rng = np.random.default_rng(31)
    shapes = [(1, 1), (1, 5), (5, 1), (31, 32), (32, 33), (33, 31), (64, 640), (513, 600),
              (1024, 1500), (1500, 1024), (2000, 2040), (7, 2000), (600, 700)]
    lens = [n for n, _ in shapes] + [m for _, m in shapes]
    p, q, off, lens = make(rng, lens)
    check(run(ffd, p, q, off, lens, "l2"), p, q, off, lens, 2, "l2")


def test_dtw_identity_and_unsupported(ffd):
    rng = np.random.default_rng(32)
    p, q, off, lens = make(rng, [50, 70, 50, 70])
    B = 2
    same_off = np.concatenate([off[:B], off[:B]])
    same_len = np.concatenate([lens[:B], lens[:B]])
    got = run(ffd, p, p, same_off, same_len, "l2")
    assert (got == 0).all()
    pi = torch.zeros((4, 2), dtype=torch.int32, device="cuda")
    o = torch.tensor([0, 2, 0, 2], dtype=torch.int64, device="cuda")
    ln = torch.tensor([2, 2, 2, 2], dtype=torch.int32, device="cuda")
    with pytest.raises(ffd.FFDError):
        ffd.dtw_batch(pi, pi, o, ln, norm="sql2")


def test_dtw_too_long_is_nan(ffd):
    """no long-pair path for DTW: documented NaN (include/ffd.h)"""
    rng = np.random.default_rng(33)
    p, q, off, lens = make(rng, [9000, 40, 9500, 50])   # 9000 rows: more than 16 bands
    got = run(ffd, p, q, off, lens, "l2")
    assert np.isnan(got[0])
    assert got[1] == oracle.dtw_pair(p[off[1]:off[1] + 40], q[off[3]:off[3] + 50], "l2", mirror=True)


def test_dtw_medium_pairs_stay_on_batch_kernel(ffd):
    """Fréchet sends pairs above 3584 rows to the long-pair kernel; DTW has no
    long-pair path, so they must stay on the batch kernel's bands (not NaN)."""
    rng = np.random.default_rng(41)
    lens = [4000, 3700, 4500, 5000]
    p, q, off, lens = make(rng, lens)
    got = run(ffd, p, q, off, lens, "sql2")
    assert np.isfinite(got).all()
    check(got, p, q, off, lens, 2, "sql2")
