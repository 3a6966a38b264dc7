"""Parity of the long-pair wavefront kernel (pairs too long for one warp band
scratch; BASELINE config 5) against the CPU oracle."""
import hashlib
import json
import os

import numpy as np
import pytest

import oracle
import workload

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

GOLD_C5 = os.path.join(os.path.dirname(__file__), "golden", "c5_expected.json")


@pytest.fixture(scope="module")
def ffd():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2404_05708_b200 as ffd
    ffd.lib()
    return ffd


def walk(rng, n, dim=2, kind="f", step=1):
    if kind == "i":
        return np.cumsum(rng.integers(-step, step + 1, size=(n, dim)), axis=0).astype(np.int32)
    return np.cumsum(rng.normal(size=(n, dim)), axis=0).astype(np.float32)


def run_pairs(ffd, pairs, norm):
    P = np.concatenate([p for p, _ in pairs])
    Q = np.concatenate([q for _, q in pairs])
    lp = np.array([len(p) for p, _ in pairs], np.int32)
    lq = np.array([len(q) for _, q in pairs], np.int32)
    op = np.concatenate([[0], np.cumsum(lp)[:-1]]).astype(np.int64)
    oq = np.concatenate([[0], np.cumsum(lq)[:-1]]).astype(np.int64)
    args = [torch.from_numpy(a).cuda() for a in (P, Q, np.concatenate([op, oq]), np.concatenate([lp, lq]))]
    return ffd.batch(*args, norm=norm).cpu().numpy()


@pytest.mark.parametrize("norm", ["l2", "l1", "linf"])
def test_long_pairs_f32(ffd, norm):
    rng = np.random.default_rng(3)
    shapes = [(600, 5000), (5000, 6000), (3000, 3000), (7000, 600), (40, 70)]
    pairs = [(walk(rng, n), walk(rng, m)) for n, m in shapes]
    got = run_pairs(ffd, pairs, norm)
    for k, (p, q) in enumerate(pairs):
        ref = oracle.pair(p, q, norm, form="linear")
        mir = oracle.pair(p, q, norm, form="mirror")
        assert abs(got[k] - ref) <= 1e-5 * abs(ref), (k, got[k], ref)
        assert got[k] == mir, (k, got[k], mir)


def test_long_pairs_int_exact(ffd):
    rng = np.random.default_rng(4)
    shapes = [(4000, 5000), (600, 4000)]
    pairs = [(walk(rng, n, kind="i"), walk(rng, m, kind="i")) for n, m in shapes]
    got = run_pairs(ffd, pairs, "sql2")
    for k, (p, q) in enumerate(pairs):
        assert got[k] == oracle.pair(p, q, "sql2", form="linear")


@pytest.mark.parametrize("ctas", ["3", "6", "1", "2"])
def test_long_pair_rows_per_lane(ffd, ctas):
    """Fewer CTAs force taller bands (R = 32 / 16); when even R = 32 does not fit
    every band at once (1 or 2 CTAs: 40 bands of 512 rows on 8 or 16 slots) the
    pair runs in several passes chained through the group's wrap link."""
    rng = np.random.default_rng(5)
    pairs = [(walk(rng, 20000), walk(rng, 20000)), (walk(rng, 300), walk(rng, 5000))]
    os.environ["FFD_LONG_CTAS"] = ctas
    try:
        got = run_pairs(ffd, pairs, "l2")
    finally:
        del os.environ["FFD_LONG_CTAS"]
    for k, (p, q) in enumerate(pairs):
        assert got[k] == _mirror_l2(k, p, q), k
    p, q = pairs[0]
    ref = oracle.pair(p, q, "l2", form="linear")
    assert abs(got[0] - ref) <= 1e-5 * ref


_MIRROR_CACHE = {}


def _mirror_l2(k, p, q):
    if k not in _MIRROR_CACHE:
        _MIRROR_CACHE[k] = oracle.pair(p, q, "l2", form="mirror")
    return _MIRROR_CACHE[k]


@pytest.mark.parametrize("norm", ["l1", "linf", "sql2"])
def test_multipass_groups_several_pairs(ffd, norm):
    """Several multi-pass pairs in one call on one or two CTA groups (tag bases
    advance by one stream per pass; odd stream lengths; pairs of different pass
    counts), fp32 and exact int32."""
    rng = np.random.default_rng(7)
    shapes = [(9000, 9001), (4100, 12000), (6000, 5999), (700, 20000)]
    kind = "i" if norm == "sql2" else "f"
    pairs = [(walk(rng, n, kind=kind), walk(rng, m, kind=kind)) for n, m in shapes]
    exp = [oracle.pair(p, q, norm, form="mirror" if kind == "f" else "linear") for p, q in pairs]
    for ctas in ("1", "2"):
        os.environ["FFD_LONG_CTAS"] = ctas
        try:
            got = run_pairs(ffd, pairs, norm)
        finally:
            del os.environ["FFD_LONG_CTAS"]
        for k in range(len(pairs)):
            assert got[k] == exp[k], (ctas, k, got[k], exp[k])


def test_beyond_coresident_rows_closed_form(ffd):
    """A pair longer than every band the GPU holds at once (148 × 8 × 32 × 32 =
    1,212,416 rows; round 1 returned NaN): n = m = 1,250,000 under L∞ with
    q = p + t, whose δ is ‖t‖∞ exactly (the (0,0) cell forces it, the diagonal
    coupling attains it; integer coordinates are exact in fp32)."""
    rng = np.random.default_rng(8)
    n = 1_250_000
    p = np.cumsum(rng.integers(-1, 2, size=(n, 2)), axis=0).astype(np.float32)
    q = p + np.array([3.0, -4.0], np.float32)
    got = run_pairs(ffd, [(p, q)], "linf")
    assert got[0] == 4.0


@pytest.mark.parametrize("norm", ["sql2", "l1", "linf"])
def test_long_int_pairs_outside_fp32_window(ffd, norm):
    """≤ 148 int32 pairs above 512 rows (so every pair runs on the long-pair CTA
    groups) with coordinates spread over ±20000: they leave the fp32-exact window
    and must be recomputed by the exact int64 tier, bit-exact (round 1 wrote
    INT64_MIN).  Squared distances reach 3.2e9 > 2^31."""
    rng = np.random.default_rng(9)
    pairs = []
    for _ in range(40):
        n, m = (int(x) for x in rng.integers(600, 5001, size=2))
        pairs.append((rng.integers(-20000, 20001, size=(n, 2)).astype(np.int32),
                      rng.integers(-20000, 20001, size=(m, 2)).astype(np.int32)))
    # and two walks that stay inside the window (the fp32 tier result is kept)
    pairs += [(walk(rng, 3000, kind="i"), walk(rng, 2500, kind="i")) for _ in range(2)]
    got = run_pairs(ffd, pairs, norm)
    P = np.concatenate([p for p, _ in pairs])
    Q = np.concatenate([q for _, q in pairs])
    lp = np.array([len(p) for p, _ in pairs], np.int32)
    lq = np.array([len(q) for _, q in pairs], np.int32)
    off = np.concatenate([np.concatenate([[0], np.cumsum(lp)[:-1]]),
                          np.concatenate([[0], np.cumsum(lq)[:-1]])]).astype(np.int64)
    exp = oracle.batch(P, Q, off, np.concatenate([lp, lq]), 2, norm, threads=0)
    bad = np.flatnonzero(got != exp)
    assert bad.size == 0, (bad[:5], got[bad[:5]], exp[bad[:5]])


def test_batch_int_multiband_outside_fp32_window(ffd):
    """More pairs than SMs, 600–3000 points (multi-band pairs on the batch kernel)
    with coordinates over ±20000: the batch kernel's exact int64 tier, bit-exact."""
    rng = np.random.default_rng(10)
    pairs = []
    for _ in range(200):
        n, m = (int(x) for x in rng.integers(600, 3001, size=2))
        pairs.append((rng.integers(-20000, 20001, size=(n, 3)).astype(np.int32),
                      rng.integers(-20000, 20001, size=(m, 3)).astype(np.int32)))
    got = run_pairs(ffd, pairs, "sql2")
    P = np.concatenate([p for p, _ in pairs])
    Q = np.concatenate([q for _, q in pairs])
    lp = np.array([len(p) for p, _ in pairs], np.int32)
    lq = np.array([len(q) for _, q in pairs], np.int32)
    off = np.concatenate([np.concatenate([[0], np.cumsum(lp)[:-1]]),
                          np.concatenate([[0], np.cumsum(lq)[:-1]])]).astype(np.int64)
    exp = oracle.batch(P, Q, off, np.concatenate([lp, lq]), 3, "sql2", threads=0)
    bad = np.flatnonzero(got != exp)
    assert bad.size == 0, (bad[:5], got[bad[:5]], exp[bad[:5]])


def test_config5_full_size(ffd):
    if not os.path.exists(GOLD_C5):
        pytest.skip("golden values not generated (scripts/make_golden_c5.py)")
    gold = json.load(open(GOLD_C5))
    p, q = workload.gen_long_pair(workload.CONFIGS[5])
    assert hashlib.sha256(p.tobytes() + q.tobytes()).hexdigest() == gold["input_sha256"]
    for norm, ref in gold["expected"].items():
        got = run_pairs(ffd, [(p, q)], norm)[0]
        assert abs(got - ref) <= 1e-5 * abs(ref), (norm, got, ref)


def test_many_long_pairs_in_one_call(ffd):
    """Successive long pairs whose streams are not a multiple of the link-ring size
    (regression: link slots must be indexed by absolute stream position, otherwise a
    producer already on the next pair overwrites the previous pair's last slots)."""
    rng = np.random.default_rng(6)
    shapes = [(2048, 2049)] * 12 + [(3000, 2600), (2047, 2100), (5000, 4099)]
    pairs = [(walk(rng, n), walk(rng, m)) for n, m in shapes]
    got = run_pairs(ffd, pairs, "l2")
    for k, (p, q) in enumerate(pairs):
        assert got[k] == oracle.pair(p, q, "l2", form="mirror"), k


def _check_mirror_batch(got, pairs, norm):
    P = np.concatenate([p for p, _ in pairs])
    Q = np.concatenate([q for _, q in pairs])
    lp = np.array([len(p) for p, _ in pairs], np.int32)
    lq = np.array([len(q) for _, q in pairs], np.int32)
    off = np.concatenate([np.concatenate([[0], np.cumsum(lp)[:-1]]),
                          np.concatenate([[0], np.cumsum(lq)[:-1]])]).astype(np.int64)
    mir = oracle.batch(P, Q, off, np.concatenate([lp, lq]), P.shape[1], norm, mirror=True)
    bad = np.flatnonzero(got != mir)
    assert bad.size == 0, (bad[:5], got[bad[:5]], mir[bad[:5]])


@pytest.mark.parametrize("norm", ["l2", "linf"])
def test_medium_pairs_on_cta_groups(ffd, norm):
    """Pairs whose shorter curve exceeds 3584 points run on the long-pair kernel,
    one group of CTAs per pair, several pairs side by side (group = li mod NG)
    and several pairs in turn on one group; mixed with short pairs."""
    rng = np.random.default_rng(31)
    shapes = [(int(rng.integers(3585, 6000)), int(rng.integers(3585, 9000))) for _ in range(40)]
    shapes += [(int(rng.integers(1, 400)), int(rng.integers(1, 400))) for _ in range(20)]
    rng.shuffle(shapes)
    pairs = [(walk(rng, n), walk(rng, m)) for n, m in shapes]
    _check_mirror_batch(run_pairs(ffd, pairs, norm), pairs, norm)


def test_medium_pairs_more_than_groups(ffd):
    """300 pairs of 3600 points: 148 groups of one CTA, two or three pairs per
    group in sequence (tag bases advance per group)."""
    rng = np.random.default_rng(32)
    pairs = [(walk(rng, 3600, kind="i"), walk(rng, 3600 + k % 7, kind="i")) for k in range(300)]
    got = run_pairs(ffd, pairs, "sql2")
    _check_mirror_batch(got, pairs, "sql2")


def test_medium_pairs_multi_cta_groups(ffd):
    """three 8192-point pairs (the paper's E2 top size): groups of many CTAs,
    cluster DSMEM and L2 links inside each group"""
    rng = np.random.default_rng(33)
    pairs = [(walk(rng, 8192), walk(rng, 8192)) for _ in range(3)] + [(walk(rng, 100), walk(rng, 90))]
    _check_mirror_batch(run_pairs(ffd, pairs, "l1"), pairs, "l1")
    os.environ["FFD_LONG_CTAS"] = "5"
    try:
        _check_mirror_batch(run_pairs(ffd, pairs, "l1"), pairs, "l1")
    finally:
        del os.environ["FFD_LONG_CTAS"]


def test_small_batch_multiband_pairs_on_groups(ffd):
    """A batch of at most one pair per SM sends every pair above 512 rows to the
    CTA groups (E1 at N ≤ 128): exact against the fp32 mirror, with single-band
    pairs of the same batch staying on the batch kernel."""
    rng = np.random.default_rng(34)
    pairs = [(walk(rng, 1024), walk(rng, 1024)) for _ in range(20)]
    pairs += [(walk(rng, int(rng.integers(513, 3000))), walk(rng, int(rng.integers(513, 3000)))) for _ in range(20)]
    pairs += [(walk(rng, 300), walk(rng, 2000)), (walk(rng, 40), walk(rng, 30))]
    _check_mirror_batch(run_pairs(ffd, pairs, "l2"), pairs, "l2")


def test_int64_tier_multipass(ffd):
    """An int32 pair outside the fp32-exact window on 1–2 CTAs: the exact int64
    tier runs it in several passes through the wrap link (64-bit values travel
    as two tagged slots), bit-exact; with an in-window pair beside it."""
    rng = np.random.default_rng(12)
    pairs = [(rng.integers(-20000, 20001, size=(9000, 2)).astype(np.int32),
              rng.integers(-20000, 20001, size=(8700, 2)).astype(np.int32)),
             (walk(rng, 6000, kind="i"), walk(rng, 6500, kind="i"))]
    exp = [oracle.pair(p, q, "sql2", form="linear") for p, q in pairs]
    for ctas in ("1", "2"):
        os.environ["FFD_LONG_CTAS"] = ctas
        try:
            got = run_pairs(ffd, pairs, "sql2")
        finally:
            del os.environ["FFD_LONG_CTAS"]
        assert list(got) == exp, (ctas, got, exp)
