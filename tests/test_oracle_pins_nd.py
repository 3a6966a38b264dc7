"""Pins for the oracle parts round 1 left unpinned.

  * orc_hausdorff_d: hand examples where only ONE direction of the
    discrete Hausdorff distance dominates (a version that drops either direction,
    or returns 0, fails), and an independent NumPy max-of-min on random d.
  * point distances at D = 1, 3, 4 for fp32 and int32 input (the round-1 pins
    used D = 2 only): hand examples (tests/golden/worked_examples.json
    "frechet_nd"), SciPy's cdist metrics (an independent library, which the C
    oracle does not call), the translation closed form δ(p, p+t) = ‖t‖ and brute
    force over couplings at D = 3 and 4.
  * the batch / cdist marshalling (orc_batch_f32, _f32mirror, _i32,
    _dtw_f32, _dtw_f32mirror, orc_cdist_entries_*) against per-pair calls on
    ragged, permuted, overlapping and one-vs-many layouts, including empty pairs.
"""
import json
import math
import os

import numpy as np
import pytest
from scipy.spatial.distance import cdist as scipy_cdist

import oracle

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "worked_examples.json")))
SCIPY_METRIC = {"l1": "cityblock", "l2": "euclidean", "linf": "chebyshev", "sql2": "sqeuclidean"}


def rand_curve(rng, n, dim, kind="f"):
    if kind == "i":
        return np.cumsum(rng.integers(-3, 4, size=(n, dim)), axis=0).astype(np.int32)
    return np.cumsum(rng.normal(size=(n, dim)), axis=0).astype(np.float32)


def py_brute(d):
    """Independent enumeration of monotone couplings (definition)."""
    P, Q = d.shape
    best = math.inf

    def rec(i, j, cur):
        nonlocal best
        if cur >= best:
            return
        if i == P - 1 and j == Q - 1:
            best = cur
            return
        for di, dj in ((1, 0), (0, 1), (1, 1)):
            a, b = i + di, j + dj
            if a < P and b < Q:
                rec(a, b, max(cur, d[a, b]))

    rec(0, 0, d[0, 0])
    return best


# ---------------------------------------------------------------------------
# Hausdorff (δ_dF ≥ the discrete Hausdorff distance)
# ---------------------------------------------------------------------------

def test_hausdorff_one_direction_dominates():
    # p = {(0,0)}, q = {(0,0), (10,0)}: every p point is ON q (p→q = 0), but q's
    # far point is 10 from p (q→p = 10).  Dropping the q→p direction gives 0.
    p = np.array([[0, 0]], np.float32)
    q = np.array([[0, 0], [10, 0]], np.float32)
    d = oracle.dist_matrix(p, q, "l2")
    assert oracle.hausdorff_d(d) == 10.0
    # transposed: p→q = 10, q→p = 0.  Dropping the p→q direction gives 0.
    assert oracle.hausdorff_d(d.T.copy()) == 10.0
    # both directions non-zero and different: p = {0, 4}, q = {1, 9} on a line
    # p→q = max(min(1,9), min(3,5)) = 3;  q→p = max(min(1,3), min(9,5)) = 5
    p1 = np.array([[0], [4]], np.float32)
    q1 = np.array([[1], [9]], np.float32)
    d1 = oracle.dist_matrix(p1, q1, "l1")
    assert d1.tolist() == [[1.0, 9.0], [3.0, 5.0]]
    assert oracle.hausdorff_d(d1) == 5.0
    assert oracle.hausdorff_d(d1.T.copy()) == 5.0
    # δ_dF of that pair: couplings (0,0)(1,1) → 5, (0,0)(0,1)(1,1) → 9,
    # (0,0)(1,0)(1,1) → 5; δ = 5 ≥ Hausdorff 5 (the bound is tight here)
    assert oracle.pair(p1, q1, "l1") == 5.0


def test_hausdorff_random_vs_numpy():
    rng = np.random.default_rng(31)
    for _ in range(200):
        n, m = rng.integers(1, 40, size=2)
        d = rng.exponential(size=(n, m))
        ref = max(d.min(axis=1).max(), d.min(axis=0).max())
        assert oracle.hausdorff_d(d) == ref
    # zero iff the point sets coincide
    p = rand_curve(rng, 12, 2)
    d = oracle.dist_matrix(p, p[::-1].copy(), "l2")
    assert oracle.hausdorff_d(d) == 0.0


# ---------------------------------------------------------------------------
# point distances at D = 1, 3, 4 (fp32 and int32)
# ---------------------------------------------------------------------------

@pytest.mark.parametrize("ex", GOLD["frechet_nd"], ids=lambda e: e["id"])
def test_worked_examples_nd(ex):
    for norm, expected in ex["expected"].items():
        if norm != "l2":
            p = np.array(ex["p"], np.int32)
            q = np.array(ex["q"], np.int32)
            for form in ("table", "linear"):
                assert oracle.pair(p, q, norm, form=form) == expected
                assert oracle.pair(q, p, norm, form=form) == expected
        p = np.array(ex["p"], np.float32)
        q = np.array(ex["q"], np.float32)
        for form in ("table", "linear", "mirror"):
            assert oracle.pair(p, q, norm, form=form) == expected


@pytest.mark.parametrize("dim", [1, 2, 3, 4])
def test_dist_matrix_vs_scipy(dim):
    rng = np.random.default_rng(40 + dim)
    for _ in range(20):
        n, m = rng.integers(1, 30, size=2)
        pf, qf = rand_curve(rng, n, dim), rand_curve(rng, m, dim)
        pi, qi = rand_curve(rng, n, dim, "i"), rand_curve(rng, m, dim, "i")
        for norm, metric in SCIPY_METRIC.items():
            ref = scipy_cdist(pf.astype(np.float64), qf.astype(np.float64), metric)
            got = oracle.dist_matrix(pf, qf, norm)
            np.testing.assert_allclose(got, ref, rtol=1e-14, atol=0)
            if norm != "l2":
                refi = scipy_cdist(pi.astype(np.float64), qi.astype(np.float64), metric)
                goti = oracle.dist_matrix(pi, qi, norm)
                assert goti.dtype == np.int64
                assert np.array_equal(goti, refi.astype(np.int64))


@pytest.mark.parametrize("dim", [1, 3, 4])
def test_translation_closed_form_nd(dim):
    """δ(p, p+t) = ‖t‖ for equal-length curves, every norm, int and float."""
    rng = np.random.default_rng(50 + dim)
    for _ in range(30):
        n = int(rng.integers(1, 120))
        p = rand_curve(rng, n, dim, "i")
        t = rng.integers(-40, 41, size=dim)
        q = (p + t).astype(np.int32)
        a = np.abs(t)
        assert oracle.pair(p, q, "sql2") == int((t * t).sum())
        assert oracle.pair(p, q, "l1") == int(a.sum())
        assert oracle.pair(p, q, "linf") == int(a.max())
        pf, qf = p.astype(np.float32), q.astype(np.float32)
        assert oracle.pair(pf, qf, "l2") == math.sqrt(float((t * t).sum()))
        assert oracle.pair(pf, qf, "l1") == float(a.sum())
        assert oracle.pair(pf, qf, "linf") == float(a.max())


@pytest.mark.parametrize("dim", [1, 3, 4])
def test_brute_force_nd(dim):
    """Pair-level δ (lazily evaluated d) = brute force over couplings of SciPy's
    distance matrix, D = 1, 3, 4, float and int."""
    rng = np.random.default_rng(60 + dim)
    for _ in range(300):
        n, m = rng.integers(1, 7, size=2)
        kind = "i" if rng.integers(0, 2) else "f"
        p, q = rand_curve(rng, n, dim, kind), rand_curve(rng, m, dim, kind)
        norms = ["l1", "linf", "sql2"] if kind == "i" else ["l1", "l2", "linf", "sql2"]
        norm = norms[rng.integers(0, len(norms))]
        d = scipy_cdist(p.astype(np.float64), q.astype(np.float64), SCIPY_METRIC[norm])
        ref = py_brute(d)
        got = oracle.pair(p, q, norm)
        if kind == "i":
            assert got == int(ref)
        else:
            assert got == pytest.approx(ref, rel=1e-14, abs=0)
        assert oracle.pair(p, q, norm, form="linear") == got


# ---------------------------------------------------------------------------
# batch / cdist marshalling = per-pair calls
# ---------------------------------------------------------------------------

def ragged_layout(rng, B, npts_p, npts_q, maxlen, empty=0):
    """Offsets/lengths in a permuted, overlapping, ragged layout inside point
    arrays of npts_p / npts_q points; `empty` pairs get a zero length."""
    lp = rng.integers(1, maxlen + 1, size=B)
    lq = rng.integers(1, maxlen + 1, size=B)
    op = np.array([rng.integers(0, npts_p - l + 1) for l in lp])
    oq = np.array([rng.integers(0, npts_q - l + 1) for l in lq])
    lens = np.concatenate([lp, lq]).astype(np.int32)
    for k in rng.choice(B, size=empty, replace=False):
        lens[k if rng.integers(0, 2) else B + k] = 0
    return np.concatenate([op, oq]).astype(np.int64), lens


def _pairs(p, q, offs, lens):
    B = offs.shape[0] // 2
    for k in range(B):
        yield k, p[offs[k]: offs[k] + lens[k]], q[offs[B + k]: offs[B + k] + lens[B + k]]


@pytest.mark.parametrize("dim", [1, 2, 3, 4])
def test_batch_f32_and_mirror_match_pairs(dim):
    rng = np.random.default_rng(70 + dim)
    p, q = rand_curve(rng, 300, dim), rand_curve(rng, 250, dim)
    offs, lens = ragged_layout(rng, 40, 300, 250, 60, empty=3)
    for norm in ("l1", "l2", "linf", "sql2"):
        out = oracle.batch(p, q, offs, lens, dim, norm, threads=2, check=False)
        outm = oracle.batch(p, q, offs, lens, dim, norm, threads=2, mirror=True, check=False)
        for k, pk, qk in _pairs(p, q, offs, lens):
            if len(pk) == 0 or len(qk) == 0:
                assert math.isnan(out[k]) and math.isnan(outm[k])
                continue
            assert out[k] == oracle.pair(pk, qk, norm)
            assert outm[k] == oracle.pair(pk, qk, norm, form="mirror")
    with pytest.raises(oracle.OracleError) as e:
        oracle.batch(p, q, offs, lens, dim, "l2")
    assert e.value.status == -4


@pytest.mark.parametrize("dim", [1, 3, 4])
def test_batch_i32_matches_pairs_nd(dim):
    rng = np.random.default_rng(80 + dim)
    p, q = rand_curve(rng, 300, dim, "i"), rand_curve(rng, 250, dim, "i")
    offs, lens = ragged_layout(rng, 40, 300, 250, 60, empty=2)
    for norm in ("l1", "linf", "sql2"):
        out = oracle.batch(p, q, offs, lens, dim, norm, threads=2, check=False)
        for k, pk, qk in _pairs(p, q, offs, lens):
            if len(pk) == 0 or len(qk) == 0:
                assert out[k] == np.iinfo(np.int64).min
                continue
            assert out[k] == oracle.pair(pk, qk, norm)


def test_batch_one_vs_many():
    """The paper's own layout: every q offset equal."""
    rng = np.random.default_rng(90)
    B = 25
    lp = rng.integers(1, 50, size=B)
    p = rand_curve(rng, int(lp.sum()), 2)
    q = rand_curve(rng, 37, 2)
    offs = np.concatenate([np.concatenate([[0], np.cumsum(lp)[:-1]]), np.zeros(B)]).astype(np.int64)
    lens = np.concatenate([lp, np.full(B, 37)]).astype(np.int32)
    out = oracle.batch(p, q, offs, lens, 2, "l2", threads=3)
    for k, pk, qk in _pairs(p, q, offs, lens):
        assert out[k] == oracle.pair(pk, qk, "l2")


@pytest.mark.parametrize("dim", [1, 3])
def test_batch_dtw_matches_pairs(dim):
    rng = np.random.default_rng(100 + dim)
    p, q = rand_curve(rng, 200, dim), rand_curve(rng, 180, dim)
    offs, lens = ragged_layout(rng, 30, 200, 180, 50, empty=2)
    for norm in ("l1", "l2", "linf", "sql2"):
        out = oracle.dtw_batch(p, q, offs, lens, dim, norm, threads=2, check=False)
        outm = oracle.dtw_batch(p, q, offs, lens, dim, norm, threads=2, mirror=True, check=False)
        for k, pk, qk in _pairs(p, q, offs, lens):
            if len(pk) == 0 or len(qk) == 0:
                assert math.isnan(out[k]) and math.isnan(outm[k])
                continue
            assert out[k] == oracle.dtw_pair(pk, qk, norm)
            assert outm[k] == oracle.dtw_pair(pk, qk, norm, mirror=True)


def test_cdist_entries_3d_match_pairs():
    rng = np.random.default_rng(110)
    A = np.stack([rand_curve(rng, 17, 3) for _ in range(6)])
    Bs = np.stack([rand_curve(rng, 23, 3) for _ in range(5)])
    ia = rng.integers(0, 6, size=40)
    ib = rng.integers(0, 5, size=40)
    for norm in ("l1", "l2", "linf"):
        out = oracle.cdist_entries(A, Bs, ia, ib, norm, threads=2)
        outm = oracle.cdist_entries(A, Bs, ia, ib, norm, mirror=True)
        for k in range(len(ia)):
            assert out[k] == oracle.pair(A[ia[k]], Bs[ib[k]], norm)
            assert outm[k] == oracle.pair(A[ia[k]], Bs[ib[k]], norm, form="mirror")
