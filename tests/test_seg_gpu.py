"""Parity of the segmented two-column batch kernel (csrc/seg.cuh) against the CPU oracle.

The segmented kernel takes the single-band Fréchet pairs (longer curve ≤ 512 points,
period H ≥ W + 32) of batches above 4096 pairs for every 2-D cell (exact-integer
sq-L2 / L1 / L∞, fp32 L2 / sq-L2 / L1 / L∞) and the 3-D fp32 L2 / sq-L2 cells.  Integer results must be bit-exact
against the exact int64 oracle; fp32 results bit-exact against the oracle's fp32
mirror and within 1e-5 relative of the fp64 oracle.  Shapes cover every (W, R)
shape, the period limit, items with missing pairs (counts not a multiple of G·L),
and pairs leaving the fp32-exact integer window (recomputed by the int64 tier).
"""
import numpy as np
import pytest

import oracle
import workload

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

TOL = 1e-5
B_MIN = 4097  # batches above 4096 pairs take the general prep path (the segmented kernel)


@pytest.fixture(scope="module")
def ffd():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2404_05708_b200 as ffd
    ffd.lib()
    return ffd


def to_dev(b):
    return tuple(torch.from_numpy(a).to("cuda") for a in (b.p, b.q, b.offsets, b.lengths))


def batch_from_lens(rng, lens, dim=2, kind="f", scale=1.0):
    B = len(lens) // 2
    off = np.zeros(2 * B, np.int64)
    off[1:B] = np.cumsum(lens[:B - 1])
    off[B + 1:] = np.cumsum(lens[B:-1])
    np_, nq = int(lens[:B].sum()), int(lens[B:].sum())
    if kind == "i":
        p = (np.cumsum(rng.integers(-8, 9, size=(np_, dim)), axis=0) * scale).astype(np.int32)
        q = (np.cumsum(rng.integers(-8, 9, size=(nq, dim)), axis=0) * scale).astype(np.int32)
    else:
        p = np.cumsum(rng.normal(size=(np_, dim)), axis=0).astype(np.float32)
        q = np.cumsum(rng.normal(size=(nq, dim)), axis=0).astype(np.float32)
    return workload.Batch(p, q, off, lens.astype(np.int32), dim, "l2")


def check_int(got, b, norm):
    ref = oracle.batch(b.p, b.q, b.offsets, b.lengths, b.dim, norm)
    mism = np.asarray(got) != ref
    assert not mism.any(), f"{mism.sum()} mismatches; first {np.nonzero(mism)[0][:5]}"


def check_float(got, b, norm):
    got = np.asarray(got)
    ref = oracle.batch(b.p, b.q, b.offsets, b.lengths, b.dim, norm)
    mir = oracle.batch(b.p, b.q, b.offsets, b.lengths, b.dim, norm, mirror=True)
    bad = np.abs(got.astype(np.float64) - ref) > TOL * np.abs(ref)
    assert not bad.any(), f"{bad.sum()} pairs beyond 1e-5 rel; first {np.nonzero(bad)[0][:5]}"
    mism = got != mir
    assert not mism.any(), f"{mism.sum()} pairs differ from the fp32 mirror; first {np.nonzero(mism)[0][:5]}"


def test_config2_shape_exact(ffd):
    """config 2's distribution (int32 2-D, lengths U[128, 512], sq-L2) at 6000 pairs."""
    b = workload.gen_batch(workload.CONFIGS[2].scaled(pairs=6000))
    check_int(ffd.batch(*to_dev(b), norm="sql2").cpu().numpy(), b, "sql2")


@pytest.mark.parametrize("norm", ["l2", "sql2"])
def test_random_lengths_f32(ffd, norm):
    """lengths 1..600: segmented pairs mixed with pairs of the batch kernel."""
    rng = np.random.default_rng(31 + len(norm))
    lens = rng.integers(1, 601, size=2 * 5000)
    b = batch_from_lens(rng, lens)
    check_float(ffd.batch(*to_dev(b), norm=norm).cpu().numpy(), b, norm)


def test_every_shape_and_period_edge(ffd):
    """rows at every (W, R) boundary (32·k, 32·k + 1, 256, 257, 512) and columns at the
    period limit H = W + 32 (94 / 126 columns) and one below it; both orientations."""
    rng = np.random.default_rng(41)
    rows = [1, 2, 31, 32, 33, 64, 65, 96, 97, 128, 129, 160, 192, 224, 255, 256, 257, 288, 289, 320,
            352, 384, 416, 448, 480, 511, 512]
    cols = [93, 94, 95, 125, 126, 127, 128, 200, 257, 511, 512]
    pairs = [(r, c) for r in rows for c in cols if c <= max(r, c)]
    reps = int(np.ceil(B_MIN / len(pairs)))
    nm = np.array(pairs * reps)
    flip = rng.random(len(nm)) < 0.5
    n = np.where(flip, nm[:, 1], nm[:, 0])
    m = np.where(flip, nm[:, 0], nm[:, 1])
    b = batch_from_lens(rng, np.concatenate([n, m]))
    check_float(ffd.batch(*to_dev(b), norm="l2").cpu().numpy(), b, "l2")
    bi = batch_from_lens(rng, np.concatenate([n, m]), kind="i")
    check_int(ffd.batch(*to_dev(bi), norm="sql2").cpu().numpy(), bi, "sql2")


@pytest.mark.parametrize("B", [B_MIN, 4099, 4103, 5001])
def test_uniform_shape_partial_items(ffd, B):
    """one bin only; B not a multiple of the item size (segments with a missing pair)."""
    rng = np.random.default_rng(B)
    lens = np.concatenate([np.full(B, 384), np.full(B, 250)])
    b = batch_from_lens(rng, lens, kind="i")
    check_int(ffd.batch(*to_dev(b), norm="sql2").cpu().numpy(), b, "sql2")
    lens = np.concatenate([np.full(B, 100), np.full(B, 200)])  # W = 16 (two segments)
    b = batch_from_lens(rng, lens)
    check_float(ffd.batch(*to_dev(b), norm="l2").cpu().numpy(), b, "l2")


def test_int_outside_window_exact(ffd):
    """segmented pairs whose points leave the fp32-exact window go to the int64 tier."""
    rng = np.random.default_rng(51)
    lens = rng.integers(128, 513, size=2 * 5000)
    b = batch_from_lens(rng, lens, kind="i", scale=300.0)
    b.p[: b.p.shape[0] // 2] //= 300  # half the rows curves stay inside the window
    check_int(ffd.batch(*to_dev(b), norm="sql2").cpu().numpy(), b, "sql2")


def test_identity_and_translation(ffd):
    """δ(p, p) = 0 and δ(p, p + t) = ‖t‖² (sq-L2, equal lengths) on segmented pairs."""
    rng = np.random.default_rng(61)
    B = 5000
    lens = rng.integers(96, 513, size=B)
    b = batch_from_lens(rng, np.concatenate([lens, lens]), kind="i")
    B_ = b.num_pairs
    same = workload.Batch(b.p, b.p, np.concatenate([b.offsets[:B_]] * 2),
                          np.concatenate([b.lengths[:B_]] * 2), 2, "sql2")
    assert (ffd.batch(*to_dev(same), norm="sql2").cpu().numpy() == 0).all()
    t = np.array([3, -4], np.int32)
    shifted = workload.Batch(b.p, b.p + t, np.concatenate([b.offsets[:B_]] * 2),
                             np.concatenate([b.lengths[:B_]] * 2), 2, "sql2")
    assert (ffd.batch(*to_dev(shifted), norm="sql2").cpu().numpy() == 25).all()


@pytest.mark.parametrize("norm", ["l1", "linf"])
def test_l1_linf_f32_and_int(ffd, norm):
    """the 2-D L1 / L∞ cells (fp32: bit-exact vs the mirror; int32: exact, also outside the window)."""
    rng = np.random.default_rng(71 + len(norm))
    lens = rng.integers(1, 601, size=2 * 4500)
    b = batch_from_lens(rng, lens)
    check_float(ffd.batch(*to_dev(b), norm=norm).cpu().numpy(), b, norm)
    bi = batch_from_lens(rng, lens, kind="i")
    check_int(ffd.batch(*to_dev(bi), norm=norm).cpu().numpy(), bi, norm)
    bw = batch_from_lens(rng, lens, kind="i", scale=20000.0)
    bw.p[: bw.p.shape[0] // 2] //= 20000
    check_int(ffd.batch(*to_dev(bw), norm=norm).cpu().numpy(), bw, norm)


@pytest.mark.parametrize("norm", ["l2", "sql2"])
def test_3d_f32(ffd, norm):
    """the 3-D fp32 L2 / sq-L2 cell (config 3's dimension), lengths 1..700."""
    rng = np.random.default_rng(81 + len(norm))
    lens = rng.integers(1, 701, size=2 * 4300)
    b = batch_from_lens(rng, lens, dim=3)
    check_float(ffd.batch(*to_dev(b), norm=norm).cpu().numpy(), b, norm)
