"""The seeded Kronecker input generator (paper_1408_1605_b200/inputs): contract checks."""
import numpy as np
import pytest

from paper_1408_1605_b200 import inputs


def test_counts_and_range():
    for scale in (0, 1, 3, 10):
        s, d = inputs.generate(scale, edgefactor=2)
        assert s.size == d.size == 2 << scale  # M = ef * 2^scale
        assert int(s.max()) < (1 << scale) and int(d.max()) < (1 << scale)
    s, d = inputs.generate(0, edgefactor=1)
    assert s.tolist() == [0] and d.tolist() == [0]  # S:44 only the self-loop exists


def test_deterministic_and_sliceable():
    a = inputs.generate(10, seed=42)
    b = inputs.generate(10, seed=42)
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])
    c = inputs.generate(10, seed=42, k0=1000, count=777)
    assert np.array_equal(a[0][1000:1777], c[0]) and np.array_equal(a[1][1000:1777], c[1])
    e = inputs.generate(10, seed=43)
    assert not np.array_equal(a[0], e[0])
    u = inputs.generate(10, seed=42, dtype=np.uint32)
    assert np.array_equal(u[0].astype(np.uint64), a[0])


@pytest.mark.parametrize("scale", [1, 2, 5, 8, 13])
def test_scramble_is_bijection(scale):
    n = 1 << scale
    img = {inputs.scramble(scale, 7, x) for x in range(n)}
    assert img == set(range(n))


def test_thresholds():
    t = inputs.thresholds()
    assert t[0] == int(0.76 * 2**32)
    assert t[1] == int(0.57 / 0.76 * 2**32)
    assert t[2] == int(0.19 / 0.24 * 2**32)


def test_rmat_bit_statistics():
    # Unscrambled bits are not observable, but the degree skew is: R-MAT concentrates
    # endpoints. Check the quadrant probability through popcounts of the inverse-free
    # statistic: fraction of self-loops ~ sum_q p_q^2 per bit... use the max degree instead.
    s, d = inputs.generate(14)
    n = 1 << 14
    deg = np.bincount(s.astype(np.int64), minlength=n) + np.bincount(d.astype(np.int64), minlength=n)
    # heavy tail: max degree far above mean (32), many isolated vertices (~25-30% at s14-16)
    assert deg.max() > 50 * deg.mean()
    iso = float(np.mean(deg == 0))
    assert 0.15 < iso < 0.40


def test_root_sampler():
    s, d = inputs.generate(10)
    n = 1 << 10
    elig = inputs.nonisolated_mask(n, s, d)
    roots = inputs.sample_roots(n, 64, elig)
    assert len(roots) == 64 and len(set(roots)) == 64
    assert all(elig[r] for r in roots)
    assert roots == inputs.sample_roots(n, 64, lambda v: bool(elig[v]))
    # self-loop-only vertices are not eligible
    m = inputs.nonisolated_mask(4, np.array([0, 1]), np.array([0, 2]))
    assert m.tolist() == [False, True, True, False]
