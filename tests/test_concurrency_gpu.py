"""include/ffd.h promises reentrant, thread-safe, stream-ordered calls: several
streams at once (batch kernels, long-pair cooperative grids, cdist) and several
host threads in ffd_batch_host give the same results as one call at a time."""
import threading

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


def _batch(seed, with_long):
    rng = np.random.default_rng(seed)
    B = 300
    lens = rng.integers(1, 400, size=2 * B).astype(np.int32)
    if with_long:
        lens[7], lens[B + 7] = 700, 9000     # long-pair kernel
        lens[9], lens[B + 9] = 4000, 4100    # medium: CTA groups
    off = np.zeros(2 * B, np.int64)
    off[1:B] = np.cumsum(lens[:B - 1])
    off[B + 1:] = np.cumsum(lens[B:-1])
    p = np.cumsum(rng.normal(size=(int(lens[:B].sum()), 2)), 0).astype(np.float32)
    q = np.cumsum(rng.normal(size=(int(lens[B:].sum()), 2)), 0).astype(np.float32)
    return p, q, off, lens


def test_many_streams_at_once(ffd):
    cases = [_batch(s, with_long=(s % 2 == 0)) for s in range(6)]
    dev = [[torch.from_numpy(a).cuda() for a in c] for c in cases]
    ref = [ffd.batch(*d, norm="l2").cpu().numpy() for d in dev]     # one at a time
    streams = [torch.cuda.Stream() for _ in cases]
    outs = []
    torch.cuda.synchronize()
    for d, st in zip(dev, streams):
        with torch.cuda.stream(st):
            outs.append(ffd.batch(*d, norm="l2", stream=st))
    A = torch.from_numpy(np.cumsum(np.random.default_rng(1).normal(size=(64, 100, 2)), 1).astype(np.float32)).cuda()
    with torch.cuda.stream(streams[0]):
        D = ffd.cdist(A, A, norm="l2", stream=streams[0])
    torch.cuda.synchronize()
    for k in range(len(cases)):
        assert np.array_equal(outs[k].cpu().numpy(), ref[k]), k
    assert torch.equal(D, ffd.cdist(A, A, norm="l2"))
    p, q, off, lens = cases[0]
    mir = oracle.batch(p, q, off, lens, 2, "l2", mirror=True)
    assert np.array_equal(ref[0], mir)


def test_host_calls_from_threads(ffd):
    cases = [_batch(10 + s, with_long=(s == 1)) for s in range(4)]
    ref = [ffd.batch_host(*c, norm="l1") for c in cases]
    got = [None] * len(cases)
    errs = []

    def work(k):
        try:
            st = torch.cuda.Stream()
            for _ in range(3):
                got[k] = ffd.batch_host(*cases[k], norm="l1", stream=st)
        except Exception as e:  # pragma: no cover - reported below
            errs.append(repr(e))

    th = [threading.Thread(target=work, args=(k,)) for k in range(len(cases))]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert not errs, errs
    for k in range(len(cases)):
        assert np.array_equal(got[k], ref[k]), k
