"""Parity of ffd_batch (CUDA, through the C ABI) against the CPU oracle.

Integer inputs: bit-exact against the exact int64 oracle.  fp32 inputs: within
1e-5 relative of the fp64 oracle (BASELINE.json north_star) AND bit-exact
against the oracle's fp32 mirror.
"""
import numpy as np
import pytest

import oracle
import workload

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

TOL = 1e-5


@pytest.fixture(scope="module")
def ffd():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2404_05708_b200 as ffd
    ffd.lib()
    return ffd


def to_dev(b: workload.Batch):
    d = "cuda"
    return (torch.from_numpy(b.p).to(d), torch.from_numpy(b.q).to(d),
            torch.from_numpy(b.offsets).to(d), torch.from_numpy(b.lengths).to(d))


def check_float(got, b, norm, threads=0):
    ref = oracle.batch(b.p, b.q, b.offsets, b.lengths, b.dim, norm, threads=threads)
    mir = oracle.batch(b.p, b.q, b.offsets, b.lengths, b.dim, norm, threads=threads, mirror=True)
    got = np.asarray(got)
    err = np.abs(got.astype(np.float64) - ref)
    bad = err > TOL * np.abs(ref)
    assert not bad.any(), f"{bad.sum()} pairs beyond 1e-5 rel; first {np.nonzero(bad)[0][:5]} got {got[bad][:5]} ref {ref[bad][:5]}"
    mism = got != mir
    assert not mism.any(), f"{mism.sum()} pairs differ from the fp32 mirror; first {np.nonzero(mism)[0][:5]}"


def check_int(got, b, norm, threads=0):
    ref = oracle.batch(b.p, b.q, b.offsets, b.lengths, b.dim, norm, threads=threads)
    got = np.asarray(got)
    mism = got != ref
    assert not mism.any(), f"{mism.sum()} mismatches; first {np.nonzero(mism)[0][:5]} got {got[mism][:5]} ref {ref[mism][:5]}"


def make_batch(rng, B, lo, hi, dim=2, kind="f", scale=1.0, lens=None):
    if lens is None:
        lens = rng.integers(lo, hi + 1, size=2 * B).astype(np.int32)
    off = np.zeros(2 * B, np.int64)
    np_, nq = int(lens[:B].sum()), int(lens[B:].sum())
    off[1:B] = np.cumsum(lens[:B - 1])
    off[B + 1:] = np.cumsum(lens[B:-1])
    if kind == "i":
        p = np.cumsum(rng.integers(-8, 9, size=(np_, dim)), axis=0).astype(np.int32)
        q = np.cumsum(rng.integers(-8, 9, size=(nq, dim)), axis=0).astype(np.int32)
        p = (p * scale).astype(np.int32)
        q = (q * scale).astype(np.int32)
    else:
        p = (np.cumsum(rng.normal(size=(np_, dim)), axis=0) * scale).astype(np.float32)
        q = (np.cumsum(rng.normal(size=(nq, dim)), axis=0) * scale).astype(np.float32)
    return workload.Batch(p, q, off, lens, dim, "l2")


def test_config1_full(ffd):
    b = workload.gen_batch(workload.CONFIGS[1])
    out = ffd.batch(*to_dev(b), norm="l2")
    check_float(out.cpu().numpy(), b, "l2")


@pytest.mark.parametrize("lo,hi", [(1, 40), (30, 130), (100, 520), (500, 1100)])
def test_random_lengths_f32_l2(ffd, lo, hi):
    rng = np.random.default_rng(lo * 7 + hi)
    b = make_batch(rng, 300, lo, hi)
    out = ffd.batch(*to_dev(b), norm="l2")
    check_float(out.cpu().numpy(), b, "l2")


def test_config2_subset_exact(ffd):
    cfg = workload.CONFIGS[2].scaled(pairs=4000)
    b = workload.gen_batch(cfg)
    out = ffd.batch(*to_dev(b), norm="sql2")
    check_int(out.cpu().numpy(), b, "sql2")


@pytest.mark.parametrize("lo,hi", [(1, 40), (100, 600), (480, 1100)])
def test_random_int_exact(ffd, lo, hi):
    rng = np.random.default_rng(lo + hi)
    b = make_batch(rng, 300, lo, hi, kind="i")
    out = ffd.batch(*to_dev(b), norm="sql2")
    check_int(out.cpu().numpy(), b, "sql2")


def test_int_outside_fp32_window_uses_exact_tier(ffd):
    """coordinates far beyond ±1448 (the fp32-exact window) must stay exact."""
    rng = np.random.default_rng(5)
    b = make_batch(rng, 200, 1, 300, kind="i", scale=5000.0)
    # mix: half the pairs in-window, half out
    b.p[: b.p.shape[0] // 3] //= 5000
    out = ffd.batch(*to_dev(b), norm="sql2")
    check_int(out.cpu().numpy(), b, "sql2")


def test_edge_lengths(ffd):
    rng = np.random.default_rng(9)
    lens = np.array([1, 1, 2, 64, 513, 1, 33, 32, 31, 600,
                     1, 7, 1, 64, 1, 700, 32, 33, 31, 599], np.int32)
    b = make_batch(rng, 10, 0, 0, lens=lens)
    out = ffd.batch(*to_dev(b), norm="l2")
    check_float(out.cpu().numpy(), b, "l2")


def test_empty_pair_gets_nan(ffd):
    rng = np.random.default_rng(10)
    lens = np.array([5, 0, 6, 7, 3, 4], np.int32)
    b = make_batch(rng, 3, 0, 0, lens=lens)
    with pytest.raises(ffd.FFDError) as e:     # the binding validates by default
        ffd.batch(*to_dev(b), norm="l2")
    assert e.value.status == -4
    out = ffd.batch(*to_dev(b), norm="l2", validate=False).cpu().numpy()
    assert np.isnan(out[1])
    ok = [0, 2]
    for k in ok:
        B = 3
        pk = b.p[b.offsets[k]: b.offsets[k] + b.lengths[k]]
        qk = b.q[b.offsets[B + k]: b.offsets[B + k] + b.lengths[B + k]]
        assert out[k] == oracle.pair(pk, qk, "l2", form="mirror")


def test_identity_and_symmetry(ffd):
    rng = np.random.default_rng(11)
    b = make_batch(rng, 100, 1, 400)
    B = b.num_pairs
    # q := p  -> δ = 0
    same = workload.Batch(b.p, b.p, np.concatenate([b.offsets[:B], b.offsets[:B]]),
                          np.concatenate([b.lengths[:B], b.lengths[:B]]), 2, "l2")
    out = ffd.batch(*to_dev(same), norm="l2").cpu().numpy()
    assert (out == 0).all()
    # swap p and q -> identical bits
    sw = workload.Batch(b.q, b.p, np.concatenate([b.offsets[B:], b.offsets[:B]]),
                        np.concatenate([b.lengths[B:], b.lengths[:B]]), 2, "l2")
    o1 = ffd.batch(*to_dev(b), norm="l2").cpu().numpy()
    o2 = ffd.batch(*to_dev(sw), norm="l2").cpu().numpy()
    assert np.array_equal(o1, o2)


@pytest.mark.parametrize("dim", [1, 2, 3, 4])
@pytest.mark.parametrize("norm", ["l1", "l2", "linf", "sql2"])
def test_all_norms_dims_f32(ffd, norm, dim):
    rng = np.random.default_rng(100 + dim * 7 + len(norm))
    b = make_batch(rng, 150, 1, 700, dim=dim)
    out = ffd.batch(*to_dev(b), norm=norm)
    check_float(out.cpu().numpy(), b, norm)


@pytest.mark.parametrize("dim", [1, 2, 3, 4])
@pytest.mark.parametrize("norm", ["l1", "linf", "sql2"])
def test_all_norms_dims_int(ffd, norm, dim):
    rng = np.random.default_rng(200 + dim * 7 + len(norm))
    b = make_batch(rng, 150, 1, 700, dim=dim, kind="i")
    out = ffd.batch(*to_dev(b), norm=norm)
    check_int(out.cpu().numpy(), b, norm)
    # and outside the fp32-exact window (exact int64 tier)
    b2 = make_batch(rng, 60, 1, 300, dim=dim, kind="i", scale=20000.0)
    out2 = ffd.batch(*to_dev(b2), norm=norm)
    check_int(out2.cpu().numpy(), b2, norm)


def test_validate(ffd):
    rng = np.random.default_rng(12)
    b = make_batch(rng, 20, 1, 50)
    args = to_dev(b)
    assert ffd.validate(*args) == 0
    bad = args[0].clone()
    bad[3, 1] = float("nan")
    assert ffd.validate(bad, *args[1:]) == -5
    lens = args[3].clone()
    lens[2] = 0
    assert ffd.validate(args[0], args[1], args[2], lens) == -4
    offs = args[2].clone()
    offs[25] = 10**9
    assert ffd.validate(args[0], args[1], offs, args[3]) == -7
    bi = make_batch(rng, 5, 1, 20, kind="i")
    ai = to_dev(bi)
    assert ffd.validate(*ai) == 0
    big_p, big_q = ai[0].clone(), ai[1].clone()
    big_p[0, :] = 2**31 - 1          # first point of pair 0's p
    big_q[0, :] = -(2**31)           # first point of pair 0's q
    assert ffd.validate(big_p, big_q, ai[2], ai[3]) == -6


def test_batch_host_matches_device(ffd):
    cfg = workload.CONFIGS[2].scaled(pairs=500)
    b = workload.gen_batch(cfg)
    dev = ffd.batch(*to_dev(b), norm="sql2").cpu().numpy()
    host = ffd.batch_host(b.p, b.q, b.offsets, b.lengths, norm="sql2")
    assert np.array_equal(dev, host)


def test_config2_full_size_exact(ffd):
    """Full BASELINE config 2 (100k pairs, lengths U[128,512], int32 sq-L2) in the
    launch configuration bench.py times: every pair bit-exact against the int64 oracle."""
    b = workload.gen_batch(workload.CONFIGS[2])
    out = ffd.batch(*to_dev(b), norm="sql2")
    check_int(out.cpu().numpy(), b, "sql2")


def test_config3_full_size_sampled(ffd):
    """Full BASELINE config 3 (1M pairs, 3-D fp32, lengths U[256,1024], ≈15 GB of
    points) in the bench launch shape; 3000 seeded pairs checked one by one against
    the fp64 oracle (≤ 1e-5) and the fp32 mirror (bit-exact); every output finite."""
    cfg = workload.CONFIGS[3]
    b = workload.gen_batch(cfg)
    out = ffd.batch(*to_dev(b), norm="l2").cpu().numpy()
    assert np.isfinite(out).all() and (out >= 0).all()
    B = b.num_pairs
    idx = np.unique(workload.sample_indices(cfg, 0, 3000, B))
    sel = [(b.p[b.offsets[k]: b.offsets[k] + b.lengths[k]],
            b.q[b.offsets[B + k]: b.offsets[B + k] + b.lengths[B + k]]) for k in idx]
    lp = np.array([len(p) for p, _ in sel], np.int32)
    lq = np.array([len(q) for _, q in sel], np.int32)
    sub = workload.Batch(np.concatenate([p for p, _ in sel]), np.concatenate([q for _, q in sel]),
                         np.concatenate([np.concatenate([[0], np.cumsum(lp)[:-1]]),
                                         np.concatenate([[0], np.cumsum(lq)[:-1]])]).astype(np.int64),
                         np.concatenate([lp, lq]), 3, "l2")
    check_float(out[idx], sub, "l2")


@pytest.mark.parametrize("norm", ["l2", "l1"])
def test_odd_even_columns_and_bands(ffd, norm):
    """Column counts of both parities (the stream repeats the last column of pairs
    with an odd m + 1) across every band shape: 1..4 bands, R at its extremes."""
    rng = np.random.default_rng(77)
    rows = [1, 2, 31, 32, 33, 63, 64, 65, 511, 512, 513, 1023, 1024, 1025, 2047, 2048]
    lens = []
    for n in rows:
        for m in (n, n + 1, n + 2, 2000, 2001):
            lens.append((n, m))
    lens = np.array(lens, np.int32)
    L = np.concatenate([lens[:, 0], lens[:, 1]]).astype(np.int32)
    b = make_batch(rng, len(lens), 0, 0, lens=L)
    out = ffd.batch(*to_dev(b), norm=norm)
    check_float(out.cpu().numpy(), b, norm)


@pytest.mark.parametrize("B", [4096, 4097])
def test_prep_small_and_general_paths_agree(ffd, B):
    """B ≤ 4096 takes the one-block preparation kernel, larger batches the
    memset + three-kernel counting sort: both exact against the oracle, with
    empty and long pairs mixed in (their dropped-pair and long-list paths)."""
    rng = np.random.default_rng(B)
    lens = rng.integers(1, 300, size=2 * B).astype(np.int32)
    lens[5] = 0                       # empty: INT64_MIN
    lens[B + 7], lens[7] = 9000, 600  # long pair: the long-pair list
    b = make_batch(rng, B, 1, 300, kind="i", lens=lens)
    got = ffd.batch(*to_dev(b), norm="sql2", validate=False).cpu().numpy()
    ref = oracle.batch(b.p, b.q, b.offsets, b.lengths, b.dim, "sql2", check=False)
    assert got[5] == np.iinfo(np.int64).min
    keep = np.arange(B) != 5
    assert np.array_equal(got[keep], ref[keep])


def test_cuda_graph_capture_replay(ffd):
    """ffd_batch is stream-capturable: one capture, then replays over new data
    written in place into the same buffers give the oracle's results."""
    rng = np.random.default_rng(11)
    b = make_batch(rng, 16, 64, 80)
    p, q, off, lens = to_dev(b)
    out = torch.empty(16, dtype=torch.float32, device="cuda")
    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(side):
        ffd.batch(p, q, off, lens, norm="l2", out=out)   # warm-up outside capture
    torch.cuda.current_stream().wait_stream(side)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        ffd.batch(p, q, off, lens, norm="l2", out=out)
    for seed in (1, 2, 3):
        b2 = make_batch(np.random.default_rng(seed), 16, 64, 80, lens=b.lengths)
        p.copy_(torch.from_numpy(b2.p))
        q.copy_(torch.from_numpy(b2.q))
        g.replay()
        torch.cuda.synchronize()
        check_float(out.cpu().numpy(), b2, "l2")


def test_batch_host_with_and_without_long_pairs(ffd):
    """ffd_batch_host skips the long-pair launch when its host lengths show no
    long pair, and runs it when one is there: both exact."""
    rng = np.random.default_rng(23)
    for long_pair in (False, True):
        lens = rng.integers(1, 200, size=2 * 8).astype(np.int32)
        if long_pair:
            lens[3], lens[8 + 3] = 700, 9000
        b = make_batch(rng, 8, 1, 200, kind="i", lens=lens)
        got = ffd.batch_host(b.p, b.q, b.offsets, b.lengths, norm="l1")
        assert np.array_equal(got, oracle.batch(b.p, b.q, b.offsets, b.lengths, b.dim, "l1"))


@pytest.mark.parametrize("layout", ["packed", "shuffled", "one_vs_many"])
def test_batch_host_pipelined_upload(ffd, layout):
    """ffd_batch_host with ≥ 64 MB of points cuts the pairs into chunks whose
    compute overlaps the upload of the next points: exact against the device
    call for packed, permuted (non-monotone offsets) and one-vs-many layouts."""
    cfg = workload.CONFIGS[2].scaled(pairs=30000)
    b = workload.gen_batch(cfg)
    B = b.num_pairs
    off, lens = b.offsets.copy(), b.lengths.copy()
    if layout == "shuffled":
        perm = np.random.default_rng(1).permutation(B)
        off = np.concatenate([off[:B][perm], off[B:][perm]])
        lens = np.concatenate([lens[:B][perm], lens[B:][perm]])
    elif layout == "one_vs_many":
        m = int(lens[B])
        off[B:] = 0
        lens[B:] = m
    assert b.p.nbytes + b.q.nbytes >= 64 << 20
    host = ffd.batch_host(b.p, b.q, off, lens, norm="sql2")
    d = "cuda"
    dev = ffd.batch(torch.from_numpy(b.p).to(d), torch.from_numpy(b.q).to(d), torch.from_numpy(off).to(d),
                    torch.from_numpy(lens).to(d), norm="sql2").cpu().numpy()
    assert np.array_equal(host, dev)
    sel = np.random.default_rng(2).choice(B, 300, replace=False)
    ref = oracle.batch(b.p, b.q, np.concatenate([off[sel], off[B + sel]]),
                       np.concatenate([lens[sel], lens[B + sel]]), b.dim, "sql2")
    assert np.array_equal(host[sel], ref)


def test_strided_offsets_lengths_and_dim_check(ffd):
    """The binding makes strided offsets/lengths contiguous and rejects
    p/q of different dims before any launch."""
    rng = np.random.default_rng(14)
    b = make_batch(rng, 30, 1, 80)
    p, q, off, lens = to_dev(b)
    off2 = torch.stack([off, torch.full_like(off, 10**9)], 1).reshape(-1)[::2]   # stride 2
    lens2 = torch.stack([lens, torch.zeros_like(lens)], 1).reshape(-1)[::2]
    assert not off2.is_contiguous() and not lens2.is_contiguous()
    got = ffd.batch(p, q, off2, lens2, norm="l2").cpu().numpy()
    ref = ffd.batch(p, q, off, lens, norm="l2").cpu().numpy()
    assert np.array_equal(got, ref)
    with pytest.raises(ValueError):
        ffd.batch(p, torch.zeros((5, 3), dtype=torch.float32, device="cuda"), off, lens)


def test_l2_tiny_distances_exact(ffd):
    """The final square root (sqrt_result: no call, tiny inputs scaled by 2^100)
    is correctly rounded down to denormal squared distances: bit-exact against
    the fp32 mirror (C sqrtf), and within 1e-5 of the fp64 oracle wherever the
    squared distance is a normal fp32 number."""
    vals = [1e-20, 3e-22, 7e-19, 1.5e-25, 2e-30, 0.0, 1e-3]
    pairs = [(np.array([[0.0, 0.0], [1.0, 1.0]], np.float32), np.array([[v, 0.0], [1.0, 1.0]], np.float32))
             for v in vals]
    P = np.concatenate([p for p, _ in pairs])
    Q = np.concatenate([q for _, q in pairs])
    B = len(pairs)
    off = np.concatenate([np.arange(B) * 2, np.arange(B) * 2]).astype(np.int64)
    lens = np.full(2 * B, 2, np.int32)
    dev = [torch.from_numpy(a).cuda() for a in (P, Q, off, lens)]
    got = ffd.batch(*dev, norm="l2").cpu().numpy()
    mir = oracle.batch(P, Q, off, lens, 2, "l2", mirror=True)
    ref = oracle.batch(P, Q, off, lens, 2, "l2")
    assert np.array_equal(got, mir), (got, mir)
    # the 1e-5 bound of reading 10 needs the squared distance in fp32's normal
    # range: a point distance below 2^-63 (≈ 1.1e-19) squares into denormals or
    # underflows to 0 (reading 10); above it the bound holds
    normal = ref >= 2.0 ** -63
    assert np.all(np.abs(got - ref)[normal] <= 1e-5 * np.abs(ref[normal])), (got, ref)
    assert got[vals.index(0.0)] == 0.0


def _raw_batch(ffd, p, q, off, lens, norm):
    """ffd_batch itself (no point counts): the launch chain always ends with the long-pair kernel."""
    B = off.numel() // 2
    dt = 1 if p.dtype == torch.int32 else 0
    out = torch.empty(B, dtype=torch.int64 if dt else torch.float32, device=p.device)
    ws = torch.empty(int(ffd.lib().ffd_batch_workspace_bytes(B)), dtype=torch.uint8, device=p.device)
    norms = {"l1": 1, "l2": 2, "linf": 3, "sql2": 4}
    rc = ffd.lib().ffd_batch(p.data_ptr(), q.data_ptr(), off.data_ptr(), lens.data_ptr(), B, p.shape[1],
                             norms[norm], dt, out.data_ptr(), ws.data_ptr(), ws.numel(),
                             torch.cuda.current_stream().cuda_stream)
    assert rc == 0
    return out


@pytest.mark.parametrize("case", ["c1_bounded", "long_default", "long_bound_broken"])
def test_batch_maxlen_skips_long_launch(ffd, case):
    """ffd_batch_maxlen (what batch() calls): config 1 with its length bounds runs
    one kernel fewer than ffd_batch, bit-identical; with the default bounds (the
    point counts) a long pair still runs the long-pair kernel, exact vs the
    oracle; a long pair that breaks a bound ruling that kernel out gets
    INT64_MIN, the other pairs stay exact."""
    rng = np.random.default_rng(29)
    if case == "c1_bounded":
        b = workload.gen_batch(workload.CONFIGS[1])
        norm, max_len = "l2", (64, 80)
        assert b.lengths[:16].max() <= 64 and b.lengths[16:].max() <= 80
    else:
        lens = rng.integers(1, 200, size=2 * 8).astype(np.int32)
        lens[3], lens[8 + 3] = 700, 9000
        b = make_batch(rng, 8, 1, 200, kind="i", lens=lens)
        norm, max_len = "l1", (None if case == "long_default" else (200, 200))
    p, q, off, lens = to_dev(b)
    torch.cuda.synchronize()
    ffd.launches_taken()
    raw = _raw_batch(ffd, p, q, off, lens, norm)
    n_raw = ffd.launches_taken()
    got = ffd.batch(p, q, off, lens, norm=norm, validate=False, max_len=max_len)
    n_got = ffd.launches_taken()
    torch.cuda.synchronize()
    if case == "c1_bounded":
        assert n_got == n_raw - 1, (n_raw, n_got)
        assert torch.equal(raw, got)
        check_float(got.cpu().numpy(), b, norm)
        return
    ref = oracle.batch(b.p, b.q, b.offsets, b.lengths, b.dim, norm)
    assert np.array_equal(raw.cpu().numpy(), ref)
    g = got.cpu().numpy()
    if case == "long_default":
        assert n_got == n_raw
        assert np.array_equal(g, ref)
    else:
        assert n_got < n_raw
        assert g[3] == np.iinfo(np.int64).min
        keep = np.arange(8) != 3
        assert np.array_equal(g[keep], ref[keep])
