"""Pins of oracle/diagnostics.py against hand computations and processes with known answers."""
import numpy as np
import pytest

from oracle import diagnostics as od


def test_rhat_hand_computation():
    # two chains of 4 draws -> four half-chains of 2 draws
    x = np.array([[0.0, 2.0, 1.0, 3.0], [4.0, 6.0, 5.0, 7.0]])
    halves = np.array([[0, 2], [1, 3], [4, 6], [5, 7]], dtype=float)
    W = np.mean([np.var(h, ddof=1) for h in halves])            # each 2.0
    Bn = np.var([h.mean() for h in halves], ddof=1)            # means 1, 2, 5, 6
    vp = 0.5 * W + Bn
    assert od.split_rhat(x) == pytest.approx(np.sqrt(vp / W), rel=1e-15)


def test_iid_chains():
    g = np.random.default_rng(0)
    x = g.normal(size=(8, 2000))
    assert abs(od.split_rhat(x) - 1.0) < 0.01
    e = od.ess(x)
    assert 0.8 * 16000 < e < 1.25 * 16000


def test_ar1_ess_matches_theory():
    """AR(1) with coefficient phi: ESS / N -> (1 - phi) / (1 + phi)."""
    g = np.random.default_rng(1)
    phi, C, S = 0.8, 8, 5000
    x = np.zeros((C, S))
    x[:, 0] = g.normal(size=C) / np.sqrt(1 - phi * phi)
    for i in range(1, S):
        x[:, i] = phi * x[:, i - 1] + g.normal(size=C)
    e = od.ess(x)
    want = C * S * (1 - phi) / (1 + phi)
    assert 0.8 * want < e < 1.25 * want


def test_unmixed_chains_flagged():
    g = np.random.default_rng(2)
    x = g.normal(size=(4, 500)) + np.arange(4)[:, None] * 2.0
    assert od.split_rhat(x) > 1.2
    # a trend inside each chain is caught by the split
    t = np.linspace(0, 3, 500)[None, :] + 0.1 * g.normal(size=(4, 500))
    assert od.split_rhat(t) > 1.2
