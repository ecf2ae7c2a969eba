"""Pins for oracle/philox.py: published known answer + distribution properties."""
import os

import numpy as np
import pytest
from scipy import stats

from oracle import philox

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def test_known_answer_vectors():
    rows = [l.split() for l in open(os.path.join(GOLD, "philox_kat.txt"))
            if l.strip() and not l.startswith("#")]
    assert rows
    for r in rows:
        c0, c1, c2, c3, k0, k1, x0, x1, x2, x3 = (int(v, 16) for v in r)
        out = philox.philox4x32_10(c0, c1, c2, c3, k0, k1)
        assert [int(o) for o in out] == [x0, x1, x2, x3]


def test_uniforms_open_interval_and_uniform():
    w = philox.words(12345, 0, 7, 3, 250000).astype(np.float64).ravel()
    u = philox.uniform01(w)
    assert u.min() > 0.0 and u.max() < 1.0
    assert stats.kstest(u, "uniform").pvalue > 1e-3
    assert abs(u.mean() - 0.5) < 5 * np.sqrt(1 / 12 / u.size)


def test_normals_moments_and_ks():
    z = philox.normals(2024, 0, 3, 1, 1_000_000)
    assert abs(z.mean()) < 5e-3
    assert abs(z.var() - 1.0) < 5e-3
    assert stats.kstest(z[:200000], "norm").pvalue > 1e-3
    # lanes of one Box-Muller pair are uncorrelated
    zz = z[: 4 * (z.size // 4)].reshape(-1, 4)
    assert abs(np.corrcoef(zz[:, 0], zz[:, 1])[0, 1]) < 6e-3


def test_streams_distinct_and_deterministic():
    a = philox.normals(5, 0, 10, 2, 64)
    np.testing.assert_array_equal(a, philox.normals(5, 0, 10, 2, 64))
    for other in (philox.normals(5, 0, 11, 2, 64), philox.normals(5, 0, 10, 3, 64),
                  philox.normals(5, 2, 10, 2, 64), philox.normals(6, 0, 10, 2, 64)):
        assert not np.any(a == other)
    # prefix property: element j depends only on (j>>2, lane), not on n
    np.testing.assert_array_equal(philox.normals(5, 0, 10, 2, 13), a[:13])
    # seed high word enters the key
    assert philox.mh_uniform(1, 0, 0) != philox.mh_uniform(1 + (1 << 32), 0, 0)


def test_counter_wraparound_inputs_are_masked():
    # counters are 32-bit: 2^32 + j aliases j (documented iter < 2^32 requirement)
    a = philox.philox4x32_10(5, 0, 7, 1, 9, 9)
    b = philox.philox4x32_10(5 + (1 << 32), 0, 7, 1, 9, 9)
    assert [int(x) for x in a] == [int(x) for x in b]
