"""Parity of ffd_batch_dtw (DTW, PAPER Appendix B, through the C ABI)
against the CPU oracle: bit-exact against the fp32 mirror of the kernels'
operation order, and within the rounding bound of an (n+m)-term fp32 sum of the
fp64 oracle."""
import os

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


def _dtw_long_check(got, p, q, off, lens, norm, transposed):
    B = len(lens) // 2
    for k in range(B):
        pk, qk = p[off[k]:off[k] + lens[k]], q[off[B + k]:off[B + k] + lens[B + k]]
        ref = oracle.dtw_pair(pk, qk, norm)
        tol = (lens[k] + lens[B + k] + 2 + 2) * 2.0 ** -24 * abs(ref)
        assert abs(got[k] - ref) <= tol, (k, got[k], ref)
        # bit-exact against the fp32 mirror in the kernel's orientation
        mir = oracle.dtw_pair(qk, pk, norm, mirror=True) if transposed[k] else oracle.dtw_pair(pk, qk, norm, mirror=True)
        assert got[k] == mir, (k, got[k], mir)


@pytest.mark.parametrize("norm", ["l2", "l1"])
def test_dtw_long_pairs(ffd, norm):
    """Pairs too long for the batch kernel's bands (more than 16 bands of 512 rows)
    run on the long-pair kernel with the DTW cell (round 1: documented NaN); the
    kernel puts the shorter curve on the rows."""
    rng = np.random.default_rng(33)
    shapes = [(9000, 9500), (9600, 9000), (40, 50), (300, 9000)]
    p, q, off, lens = make(rng, [a for a, _ in shapes] + [b for _, b in shapes])
    got = run(ffd, p, q, off, lens, norm)
    _dtw_long_check(got, p, q, off, lens, norm, [a > b for a, b in shapes])


def test_dtw_long_multipass(ffd):
    """A DTW pair on one or two CTAs: more bands than slots, several passes through
    the wrap link (rows = the longer curve)."""
    rng = np.random.default_rng(34)
    shapes = [(8300, 9001), (9100, 8200)]
    p, q, off, lens = make(rng, [a for a, _ in shapes] + [b for _, b in shapes])
    for ctas in ("1", "2"):
        os.environ["FFD_LONG_CTAS"] = ctas
        try:
            got = run(ffd, p, q, off, lens, "sql2")
        finally:
            del os.environ["FFD_LONG_CTAS"]
        _dtw_long_check(got, p, q, off, lens, "sql2", [a < b for a, b in shapes])


def test_dtw_medium_pairs_stay_on_batch_kernel(ffd):
    """Fréchet sends pairs above 3584 rows to the long-pair kernel; DTW has no
    long-pair path, so they must stay on the batch kernel's bands (not NaN)."""
    rng = np.random.default_rng(41)
    lens = [4000, 3700, 4500, 5000]
    p, q, off, lens = make(rng, lens)
    got = run(ffd, p, q, off, lens, "sql2")
    assert np.isfinite(got).all()
    check(got, p, q, off, lens, 2, "sql2")


@pytest.mark.parametrize("norm", ["sql2", "l1", "l2", "linf"])
def test_dtw_long_kernel_small_shapes(ffd, norm):
    """FFD_DTW_LONG=1 (testing) routes every DTW pair to the long-pair kernel: small
    and odd shapes (1×1, one row, one column, odd/even column counts: one or two
    leading sentinel positions) bit-exact against the fp32 mirror in the kernel's
    orientation (the shorter curve on the rows)."""
    rng = np.random.default_rng(35)
    shapes = [(1, 1), (1, 2), (2, 1), (3, 4), (4, 3), (10, 12), (40, 50), (40, 51), (200, 333), (129, 64)]
    p, q, off, lens = make(rng, [a for a, _ in shapes] + [b for _, b in shapes])
    os.environ["FFD_DTW_LONG"] = "1"
    try:
        got = run(ffd, p, q, off, lens, norm)
    finally:
        del os.environ["FFD_DTW_LONG"]
    _dtw_long_check(got, p, q, off, lens, norm, [a > b for a, b in shapes])


def run64(ffd, p, q, off, lens, norm, validate=True):
    args = [torch.from_numpy(np.ascontiguousarray(a)).cuda() for a in (p, q, off, lens)]
    return ffd.dtw_batch(*args, norm=norm, precision="f64", validate=validate).cpu().numpy()


@pytest.mark.parametrize("dim", [1, 2, 3, 4])
@pytest.mark.parametrize("norm", ["l2", "sql2", "l1", "linf"])
def test_dtw_f64_bit_exact(ffd, norm, dim):
    """ffd_batch_dtw_f64: fp64 distances in the oracle's operation order and fp64
    sums, so every result equals the fp64 oracle (orc_pair_dtw_f32) bit for bit —
    the tight tolerance the fp32 path cannot have ((n+m+D+2)·2⁻²⁴)."""
    rng = np.random.default_rng(700 + dim * 11 + len(norm))
    lens = rng.integers(1, 700, size=2 * 80)
    lens[:4] = [1, 257, 300, 1024]       # one point; more than one 256-row band (fp64 bands: R ≤ 8)
    lens[80:84] = [5, 1, 900, 333]
    p, q, off, lens = make(rng, lens, dim=dim)
    got = run64(ffd, p, q, off, lens, norm)
    ref = oracle.dtw_batch(p, q, off, lens, dim, norm)
    assert got.dtype == np.float64
    bad = np.flatnonzero(got != ref)
    assert bad.size == 0, (bad[:5], got[bad[:5]], ref[bad[:5]])


def test_dtw_f64_edges(ffd):
    rng = np.random.default_rng(36)
    p, q, off, lens = make(rng, [5, 0, 9000, 7, 6, 40, 9500, 0])
    got = run64(ffd, p, q, off, lens, "l2", validate=False)
    assert np.isnan(got[1]) and np.isnan(got[3])   # empty curves
    assert np.isnan(got[2])                        # too long for the bands: no fp64 long-pair tier
    assert got[0] == oracle.dtw_pair(p[off[0]:off[0] + 5], q[off[4]:off[4] + 6], "l2")
