"""Pins for the CPU oracle (oracle/ffd_oracle.c) against things other than itself.

Every check here is fixed by the paper or by mathematics, not by re-typing the
oracle's formula (DESIGN.md §Oracle pins):
  * the definition: brute-force enumeration of all monotone couplings;
  * hand-derived worked examples (tests/golden/worked_examples.json);
  * closed forms: length-1 curves (running max, Alg. 4), δ(p,p)=0,
    translation δ(p, p+t) = ‖t‖;
  * invariants: symmetry, reversal, repeated points (PAPER L259 footnote),
    membership δ ∈ {d_ij}, endpoint and Hausdorff lower bounds,
    triangle inequality, norm ordering, prefix semantics (L166);
  * agreement of the table, Alg. 4, Alg. 5 and the literal Alg. 2 forms;
  * plausible mistakes (dropped diag term, prefix-min misreading of L237,
    swapped min/max) are shown to FAIL these pins.
"""
import itertools
import json
import math
import os

import numpy as np
import pytest

import oracle
import workload

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "worked_examples.json")))
NORMS = ["l1", "l2", "linf", "sql2"]


def rand_curve(rng, n, dim=2, kind="f"):
    if kind == "i":
        return np.cumsum(rng.integers(-3, 4, size=(n, dim)), axis=0).astype(np.int32)
    return np.cumsum(rng.normal(size=(n, dim)), axis=0).astype(np.float32)


# ---------------------------------------------------------------------------
# worked examples
# ---------------------------------------------------------------------------

@pytest.mark.parametrize("ex", GOLD["frechet"], ids=lambda e: e["id"])
def test_worked_examples(ex):
    expected = math.sqrt(ex["expected_sqrt"]) if "expected_sqrt" in ex else ex["expected"]
    if ex["norm"] == "sql2":
        p = np.array(ex["p"], np.int32)
        q = np.array(ex["q"], np.int32)
        assert oracle.pair(p, q, "sql2") == expected
        assert oracle.pair(p, q, "sql2", form="linear") == expected
    p = np.array(ex["p"], np.float32)
    q = np.array(ex["q"], np.float32)
    for form in ("table", "linear"):
        assert oracle.pair(p, q, ex["norm"], form=form) == pytest.approx(expected, rel=1e-15, abs=0)
    assert oracle.pair(p, q, ex["norm"], form="mirror") == pytest.approx(expected, rel=1e-6)
    d = oracle.dist_matrix(p, q, ex["norm"])
    for fn in (oracle.frechet_table_d, oracle.frechet_linear_d, oracle.frechet_alg2_d,
               oracle.frechet_inplace_d, oracle.frechet_brute_d):
        assert fn(d) == pytest.approx(expected, rel=1e-15, abs=0)


@pytest.mark.parametrize("ex", GOLD["from_d"], ids=lambda e: e["id"])
def test_worked_examples_from_d(ex):
    d = np.array(ex["d"], np.float64)
    for fn in (oracle.frechet_table_d, oracle.frechet_linear_d, oracle.frechet_alg2_d,
               oracle.frechet_inplace_d, oracle.frechet_brute_d):
        assert fn(d) == ex["expected"]
    if "table_row2" in ex:
        C = oracle.full_table_d(d)
        assert list(C[2, 1:]) == ex["table_row2"]


def prefix_min_misreading(d):
    """Alg. 5 with L237 read as a sequential in-place left-to-right min (WRONG)."""
    P, Q = d.shape
    v = np.maximum.accumulate(d[0]).tolist()
    for i in range(1, P):
        for j in range(1, Q):
            v[j] = min(v[j - 1], v[j])
        v[0] = max(v[0], d[i, 0])
        for j in range(1, Q):
            v[j] = max(min(v[j - 1], v[j]), d[i, j])
    return v[-1]


def test_prefix_min_misreading_is_caught():
    ex = [e for e in GOLD["from_d"] if e["id"] == "simultaneous_min_witness"][0]
    d = np.array(ex["d"], np.float64)
    assert prefix_min_misreading(d) == ex["wrong_if_prefix_min"] != ex["expected"]


# ---------------------------------------------------------------------------
# the definition: brute force over couplings
# ---------------------------------------------------------------------------

def py_brute(d):
    """Independent Python enumeration of monotone couplings (definition)."""
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


def test_brute_force_float():
    rng = np.random.default_rng(1)
    for _ in range(1500):
        n, m = rng.integers(1, 8, size=2)
        p, q = rand_curve(rng, n), rand_curve(rng, m)
        norm = NORMS[rng.integers(0, 3)]
        d = oracle.dist_matrix(p, q, norm)
        ref = py_brute(d)
        assert oracle.frechet_brute_d(d) == ref
        assert oracle.frechet_table_d(d) == ref
        assert oracle.frechet_linear_d(d) == ref
        assert oracle.frechet_alg2_d(d) == ref
        assert oracle.frechet_inplace_d(d) == ref
        assert oracle.pair(p, q, norm) == ref
        assert oracle.pair(p, q, norm, form="linear") == ref


def test_brute_force_int():
    rng = np.random.default_rng(2)
    for _ in range(1500):
        n, m = rng.integers(1, 8, size=2)
        p, q = rand_curve(rng, n, kind="i"), rand_curve(rng, m, kind="i")
        norm = ["l1", "linf", "sql2"][rng.integers(0, 3)]
        d = oracle.dist_matrix(p, q, norm)
        ref = py_brute(d)
        assert oracle.frechet_brute_d(d.astype(np.int64)) == ref
        assert oracle.pair(p, q, norm) == ref
        assert oracle.pair(p, q, norm, form="linear") == ref


def test_table_forms_agree_larger():
    """Alg. 3 table = Alg. 4 = Alg. 5 = Alg. 2, bit for bit (selection only), P,Q up to 200."""
    rng = np.random.default_rng(3)
    for _ in range(60):
        n, m = rng.integers(1, 200, size=2)
        d = oracle.dist_matrix(rand_curve(rng, n), rand_curve(rng, m), "l2")
        t = oracle.frechet_table_d(d)
        assert oracle.frechet_linear_d(d) == t
        assert oracle.frechet_alg2_d(d) == t
        assert oracle.frechet_inplace_d(d) == t


# plausible implementation mistakes must fail the brute-force pin
def _mut_drop_diag(d):
    P, Q = d.shape
    C = np.full((P + 1, Q + 1), np.inf)
    C[0, 0] = 0
    for i in range(1, P + 1):
        for j in range(1, Q + 1):
            C[i, j] = max(min(C[i - 1, j], C[i, j - 1]), d[i - 1, j - 1])
    return C[P, Q]


def _mut_swap_minmax(d):
    P, Q = d.shape
    C = np.full((P + 1, Q + 1), -np.inf)
    C[0, 0] = 0
    for i in range(1, P + 1):
        for j in range(1, Q + 1):
            C[i, j] = min(max(C[i - 1, j], C[i - 1, j - 1], C[i, j - 1]), d[i - 1, j - 1])
    return C[P, Q]


def _mut_off_by_one(d):
    P, Q = d.shape
    C = np.full((P + 1, Q + 1), np.inf)
    C[0, 0] = 0
    for i in range(1, P + 1):
        for j in range(1, Q + 1):
            C[i, j] = max(min(C[i - 1, j], C[i - 1, j - 1], C[i, j - 1]), d[i - 1, j - 1])
    return C[P, Q - 1] if Q > 1 else C[P, Q]


@pytest.mark.parametrize("mutant", [_mut_drop_diag, _mut_swap_minmax, _mut_off_by_one, prefix_min_misreading])
def test_mutants_fail_brute_force(mutant):
    rng = np.random.default_rng(4)
    caught = 0
    for _ in range(300):
        n, m = rng.integers(2, 7, size=2)
        d = oracle.dist_matrix(rand_curve(rng, n), rand_curve(rng, m), "l2")
        if mutant(d) != py_brute(d):
            caught += 1
    assert caught > 0


# ---------------------------------------------------------------------------
# closed forms
# ---------------------------------------------------------------------------

@pytest.mark.parametrize("norm", NORMS)
def test_length_one_is_running_max(norm):
    rng = np.random.default_rng(5)
    for _ in range(50):
        m = int(rng.integers(1, 300))
        p, q = rand_curve(rng, 1), rand_curve(rng, m)
        d = oracle.dist_matrix(p, q, norm)
        assert oracle.pair(p, q, norm) == d.max()
        assert oracle.pair(q, p, norm) == d.max()


@pytest.mark.parametrize("norm", NORMS)
def test_identity(norm):
    rng = np.random.default_rng(6)
    for _ in range(20):
        p = rand_curve(rng, int(rng.integers(1, 300)))
        assert oracle.pair(p, p, norm) == 0.0
        assert oracle.pair(p, p, norm, form="mirror") == 0.0


def test_translation_closed_form():
    """δ(p, p+t) = ‖t‖ for equal-length curves: (0,0) forces ≥ ‖t‖, the diagonal attains it."""
    rng = np.random.default_rng(7)
    for _ in range(40):
        n = int(rng.integers(1, 200))
        p = rand_curve(rng, n, kind="i")
        t = rng.integers(-50, 51, size=2)
        q = (p + t).astype(np.int32)
        assert oracle.pair(p, q, "sql2") == int(t[0] ** 2 + t[1] ** 2)
        assert oracle.pair(p, q, "l1") == int(abs(t[0]) + abs(t[1]))
        assert oracle.pair(p, q, "linf") == int(max(abs(t[0]), abs(t[1])))
        pf, qf = p.astype(np.float32), q.astype(np.float32)
        assert oracle.pair(pf, qf, "l2") == math.sqrt(float(t[0] ** 2 + t[1] ** 2))


# ---------------------------------------------------------------------------
# invariants
# ---------------------------------------------------------------------------

def test_invariants_random():
    rng = np.random.default_rng(8)
    for _ in range(150):
        n, m = rng.integers(1, 120, size=2)
        p, q = rand_curve(rng, n), rand_curve(rng, m)
        for norm in NORMS:
            d = oracle.dist_matrix(p, q, norm)
            v = oracle.pair(p, q, norm)
            assert oracle.pair(q, p, norm) == v                                # symmetry
            assert oracle.pair(p[::-1], q[::-1], norm) == v                    # reversal
            assert v in set(d.ravel().tolist())                                # selection
            assert v >= max(d[0, 0], d[-1, -1])                                # endpoints
            assert v >= oracle.hausdorff_d(d)
            # any explicit coupling bounds δ from above: the "staircase" coupling
            stair = max(d[0, :].max(), d[:, -1].max())
            assert v <= stair
            # repeated points (PAPER L259 footnote)
            k = int(rng.integers(0, n))
            p2 = np.insert(p, k, p[k], axis=0)
            assert oracle.pair(p2, q, norm) == v


def test_triangle_inequality():
    rng = np.random.default_rng(9)
    for _ in range(200):
        a, b, c = (rand_curve(rng, int(rng.integers(1, 60))) for _ in range(3))
        for norm in ("l1", "l2", "linf"):
            ab, bc, ac = oracle.pair(a, b, norm), oracle.pair(b, c, norm), oracle.pair(a, c, norm)
            assert ac <= (ab + bc) * (1 + 1e-9)


def test_norm_ordering():
    """Pointwise Linf ≤ L2 ≤ L1 ≤ √D·L2 ≤ D·Linf survives the min-max DP."""
    rng = np.random.default_rng(10)
    for _ in range(100):
        p, q = rand_curve(rng, int(rng.integers(1, 80))), rand_curve(rng, int(rng.integers(1, 80)))
        li, l2, l1 = oracle.pair(p, q, "linf"), oracle.pair(p, q, "l2"), oracle.pair(p, q, "l1")
        eps = 1e-12
        assert li <= l2 * (1 + eps) and l2 <= l1 * (1 + eps)
        assert l1 <= math.sqrt(2) * l2 * (1 + eps) and math.sqrt(2) * l2 <= 2 * li * (1 + eps)
        assert oracle.pair(p, q, "sql2") == pytest.approx(l2 * l2, rel=1e-12)


def test_prefix_semantics():
    """C[α][β] = δ of the prefixes p[:α], q[:β]."""
    rng = np.random.default_rng(11)
    p, q = rand_curve(rng, 30), rand_curve(rng, 25)
    C = oracle.full_table_d(oracle.dist_matrix(p, q, "l2"))
    for a, b in itertools.product(range(1, 31, 7), range(1, 26, 6)):
        assert C[a, b] == oracle.pair(p[:a], q[:b], "l2")


def test_mirror_close_to_fp64():
    """fp32 mirror within the fp32 error bound of the fp64 oracle (reading 10)."""
    rng = np.random.default_rng(12)
    for _ in range(100):
        p, q = rand_curve(rng, int(rng.integers(1, 100))), rand_curve(rng, int(rng.integers(1, 100)))
        for norm in ("l1", "l2", "linf"):
            ref = oracle.pair(p, q, norm)
            got = oracle.pair(p, q, norm, form="mirror")
            assert abs(got - ref) <= 1e-6 * abs(ref)


# ---------------------------------------------------------------------------
# preconditions
# ---------------------------------------------------------------------------

def test_errors():
    p = np.zeros((3, 2), np.float32)
    q = np.zeros((0, 2), np.float32)
    with pytest.raises(oracle.OracleError) as e:
        oracle.pair(p, q)
    assert e.value.status == -4
    bad = p.copy()
    bad[1, 0] = np.nan
    with pytest.raises(oracle.OracleError) as e:
        oracle.pair(bad, p)
    assert e.value.status == -5
    big = np.array([[2**31 - 1, 2**31 - 1]], np.int32)
    small = np.array([[-(2**31), -(2**31)]], np.int32)
    with pytest.raises(oracle.OracleError) as e:
        oracle.pair(big, small, "sql2")
    assert e.value.status == -6
    # L1 of the same points is representable
    assert oracle.pair(big, small, "l1") == 2 * (2**32 - 1)


# ---------------------------------------------------------------------------
# batch / cdist helpers reduce to the pair function
# ---------------------------------------------------------------------------

def test_batch_matches_pairs():
    cfg = workload.CONFIGS[2].scaled(pairs=40, len_p=(1, 60), len_q=(1, 60))
    b = workload.gen_batch(cfg)
    out = oracle.batch(b.p, b.q, b.offsets, b.lengths, b.dim, "sql2", threads=2)
    B = b.num_pairs
    for k in range(B):
        pk = b.p[b.offsets[k]: b.offsets[k] + b.lengths[k]]
        qk = b.q[b.offsets[B + k]: b.offsets[B + k] + b.lengths[B + k]]
        assert out[k] == oracle.pair(pk, qk, "sql2")


def test_cdist_entries_match_pairs():
    cfg = workload.CONFIGS[4].scaled(nA=7, nB=5, length=20)
    A, Bs = workload.gen_set(cfg, "A"), workload.gen_set(cfg, "B")
    ia = np.repeat(np.arange(7), 5)
    ib = np.tile(np.arange(5), 7)
    out = oracle.cdist_entries(A, Bs, ia, ib, "l2")
    outm = oracle.cdist_entries(A, Bs, ia, ib, "l2", mirror=True)
    for k in range(len(ia)):
        assert out[k] == oracle.pair(A[ia[k]], Bs[ib[k]], "l2")
        assert outm[k] == oracle.pair(A[ia[k]], Bs[ib[k]], "l2", form="mirror")


# ---------------------------------------------------------------------------
# DTW (Appendix B) — NEXT f2 oracle
# ---------------------------------------------------------------------------

def py_dtw_brute(d):
    P, Q = d.shape
    best = math.inf

    def rec(i, j, acc):
        nonlocal best
        if i == P - 1 and j == Q - 1:
            best = min(best, acc)
            return
        for di, dj in ((1, 0), (0, 1), (1, 1)):
            a, b = i + di, j + dj
            if a < P and b < Q:
                rec(a, b, acc + d[a, b])

    rec(0, 0, d[0, 0])
    return best


def test_dtw():
    ex = GOLD["dtw"][0]
    d = oracle.dist_matrix(np.array(ex["p"], np.float32), np.array(ex["q"], np.float32), ex["norm"])
    assert oracle.dtw_table_d(d) == ex["expected"] == oracle.dtw_alg_d(d)
    rng = np.random.default_rng(13)
    for _ in range(300):
        n, m = rng.integers(1, 7, size=2)
        d = oracle.dist_matrix(rand_curve(rng, n, kind="i").astype(np.float32),
                               rand_curve(rng, m, kind="i").astype(np.float32), "l1")
        ref = py_dtw_brute(d)   # integer-valued sums: exact
        assert oracle.dtw_table_d(d) == ref
        assert oracle.dtw_alg_d(d) == ref


def test_dtw_pairs_pinned():
    """Pair-level DTW (lazily evaluated d, PAPER Appendix B) against the C brute
    force over couplings, the distance-matrix table, and closed forms; the fp32
    mirror against fp64 within the rounding bound of a (n+m)-term sum."""
    rng = np.random.default_rng(21)
    for _ in range(300):
        n, m = rng.integers(1, 7, size=2)
        p = rand_curve(rng, n).astype(np.float32)
        q = rand_curve(rng, m).astype(np.float32)
        for norm in ("l1", "l2", "linf", "sql2"):
            d = oracle.dist_matrix(p, q, norm)
            v = oracle.dtw_pair(p, q, norm)
            assert v == oracle.dtw_table_d(d)
            assert abs(v - oracle.dtw_brute_d(d)) <= 1e-12 * max(1.0, abs(v))
            assert abs(v - py_dtw_brute(d)) <= 1e-12 * max(1.0, abs(v))
            mir = oracle.dtw_pair(p, q, norm, mirror=True)
            assert abs(mir - v) <= (n + m + 4) * 2.0 ** -24 * abs(v) + 1e-30
            # symmetric measure, exactly so in the fp32 mirror as well
            assert oracle.dtw_pair(q, p, norm, mirror=True) == mir
            # DTW(p, p) = 0; DTW ≥ δ_dF (a sum along the best coupling ≥ its max)
            assert oracle.dtw_pair(p, p, norm) == 0.0
            assert v >= oracle.pair(p, q, norm) - 1e-12
    # length-1 curve: the sum of the distances to every point (a closed form)
    p = np.array([[0.5, -1.0]], np.float32)
    q = rand_curve(rng, 9).astype(np.float32)
    ref = sum(float(np.hypot(*(q[j].astype(np.float64) - p[0]))) for j in range(9))
    assert abs(oracle.dtw_pair(p, q, "l2") - ref) <= 1e-12 * ref


def test_dist_sum_pinned():
    """Σ_ij d_ij (the paper's "upper limit" baseline)
    against closed forms that a dropped term, a wrong index or a wrong norm
    breaks, and against DTW with a one-point curve (Appendix B: the only
    coupling visits every q_j once, so DTW = Σ_j d_0j)."""
    # 1-D integer walks p_i = i, q_j = j: every norm is |i − j|.
    for n in (1, 2, 7, 33):
        p = np.arange(n, dtype=np.float32)[:, None]
        s_abs = n * (n * n - 1) / 3          # Σ_{i,j<n} |i − j|
        s_sq = n * n * (n * n - 1) / 6       # Σ_{i,j<n} (i − j)²
        for norm, ref in (("l1", s_abs), ("l2", s_abs), ("linf", s_abs), ("sql2", s_sq)):
            assert oracle.dist_sum_pair(p, p, norm) == ref
    # 3-4-5 triangles: p = {(0,0)}, q_j = (3j, 4j), j < m
    for m in (1, 5, 40):
        j = np.arange(m, dtype=np.float64)
        q = np.stack([3 * j, 4 * j], 1).astype(np.float32)
        p = np.zeros((1, 2), np.float32)
        for norm, ref in (("l2", 5 * j.sum()), ("l1", 7 * j.sum()), ("linf", 4 * j.sum()),
                          ("sql2", 25 * (j * j).sum())):
            assert oracle.dist_sum_pair(p, q, norm) == ref
            assert oracle.dist_sum_pair(q, p, norm) == ref
    # unequal lengths, 1-D: p_i = i (n points), q_j = j (m points), sql2
    n, m = 5, 9
    ref = sum((i - j) ** 2 for i in range(n) for j in range(m))
    assert oracle.dist_sum_pair(np.arange(n, dtype=np.float32)[:, None],
                                np.arange(m, dtype=np.float32)[:, None], "sql2") == ref
    rng = np.random.default_rng(5)
    for _ in range(50):
        m = int(rng.integers(1, 12))
        p = rand_curve(rng, 1).astype(np.float32)
        q = rand_curve(rng, m).astype(np.float32)
        for norm in ("l1", "l2", "linf", "sql2"):
            v = oracle.dist_sum_pair(p, q, norm)
            assert abs(v - oracle.dtw_pair(p, q, norm)) <= 1e-12 * max(1.0, v)
    # batch == pairs (one-vs-many layout: every q offset 0)
    B = 6
    lens = rng.integers(1, 20, size=2 * B).astype(np.int32)
    lens[B:] = lens[B]
    P = rand_curve(rng, int(lens[:B].sum())).astype(np.float32)
    Q = rand_curve(rng, int(lens[B])).astype(np.float32)
    offs = np.concatenate([np.concatenate([[0], np.cumsum(lens[:B])[:-1]]), np.zeros(B)]).astype(np.int64)
    got = oracle.dist_sum_batch(P, Q, offs, lens, 2, "l2")
    for k in range(B):
        assert got[k] == oracle.dist_sum_pair(P[offs[k]:offs[k] + lens[k]], Q, "l2")
