"""Generator determinism and distribution shape (workload/ffd_gen.c)."""
import numpy as np

import workload


def test_deterministic_and_independent():
    cfg = workload.CONFIGS[2].scaled(pairs=200)
    a, b = workload.gen_batch(cfg), workload.gen_batch(cfg)
    assert np.array_equal(a.p, b.p) and np.array_equal(a.q, b.q)
    assert np.array_equal(a.lengths, b.lengths)
    # curve k does not depend on how many curves are generated
    small = workload.gen_batch(cfg.scaled(pairs=50))
    assert np.array_equal(small.lengths[:50], a.lengths[:50])
    assert np.array_equal(small.p, a.p[: small.p.shape[0]])


def test_config2_shape():
    cfg = workload.CONFIGS[2].scaled(pairs=2000)
    b = workload.gen_batch(cfg)
    B = b.num_pairs
    assert b.lengths.min() >= 128 and b.lengths.max() <= 512
    assert b.p.dtype == np.int32 and b.p.shape[1] == 2
    # every curve starts at the origin, steps in [-8, 8]
    for k in range(0, B, 97):
        c = b.p[b.offsets[k]: b.offsets[k] + b.lengths[k]]
        assert (c[0] == 0).all()
        st = np.diff(c, axis=0)
        assert st.min() >= -8 and st.max() <= 8
    # uniform-ish lengths, independent p and q
    assert abs(b.lengths[:B].mean() - 320) < 10
    assert abs(np.corrcoef(b.lengths[:B], b.lengths[B:])[0, 1]) < 0.1


def test_config3_start_offsets():
    cfg = workload.CONFIGS[3].scaled(pairs=3000, len_p=(2, 2), len_q=(2, 2))
    b = workload.gen_batch(cfg)
    starts = b.p[b.offsets[:3000]]
    assert abs(starts.std() - 10.0) < 0.5       # N(0, 10^2) per coordinate
    steps = b.p[b.offsets[:3000] + 1] - starts
    assert abs(steps.std() - 1.0) < 0.05


def test_unit_walk_steps():
    cfg = workload.CONFIGS[101].scaled(pairs=4, len_p=(500, 500), len_q=(500, 500))
    b = workload.gen_batch(cfg)
    st = np.diff(b.p[:500], axis=0)
    assert set(np.unique(st).tolist()) <= {-1.0, 0.0, 1.0}
