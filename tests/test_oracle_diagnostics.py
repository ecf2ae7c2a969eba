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


def test_truncation_first_odd_lag_hand_sequence():
    """BDA3 11.8 stops at the first ODD T with rho_{T+1} + rho_{T+2} < 0.  In this hand-made
    sequence the pair sum first turns negative after the EVEN lag 2 (rho_3 + rho_4 = -0.45), so a
    rule checking every lag would stop at T = 2 (sum 1.0); the odd rule checks t = 1 (rho_2 + rho_3
    = 0.3, go on) and t = 3 (rho_4 + rho_5 = -0.30, stop): sum rho_1..rho_3 = 0.6 + 0.4 - 0.1."""
    rho = np.array([1.0, 0.6, 0.4, -0.1, -0.35, 0.05, 0.02, 0.01])
    assert od.truncated_sum(rho) == pytest.approx(0.9, abs=1e-15)
    # stop at the very first odd lag: rho_2 + rho_3 < 0 -> T = 1
    assert od.truncated_sum(np.array([1.0, 0.3, -0.2, -0.1, 0.5])) == pytest.approx(0.3, abs=1e-15)
    # no odd lag qualifies -> all available lags (n - 1 = 4)
    assert od.truncated_sum(np.array([1.0, 0.5, 0.25, 0.125, 0.0625])) == pytest.approx(0.9375, abs=1e-15)
    # n = 3: rho_1 then rho_2 (no rho_3 to test against)
    assert od.truncated_sum(np.array([1.0, 0.2, 0.1])) == pytest.approx(0.3, abs=1e-15)


def test_autocorr_hand_computation():
    """Variogram autocorrelation (BDA3 11.7) on two half-chains of 3 draws, by hand:
    halves (0, 1, 3) and (1, 2, 0); W = (7/3 + 1) / 2 = 5/3, chain means 4/3, 1 -> B/n =
    (1/3)^2 / 2 = 1/18, var+ = 2/3 W + B/n = 10/9 + 1/18 = 7/6.
    V_1 = ((1)^2 + (2)^2 + (1)^2 + (-2)^2) / (2 * 2) = 10/4; rho_1 = 1 - V_1 / (2 var+) = 1 - 15/14.
    V_2 = ((3)^2 + (-1)^2) / (2 * 1) = 5; rho_2 = 1 - 5 / (7/3) = -8/7."""
    x = np.array([[0.0, 1.0, 3.0, 1.0, 2.0, 0.0]])   # one chain of 6 draws -> halves of 3
    rho = od.autocorr(od.split_chains(x))
    np.testing.assert_allclose(rho, [1.0, 1.0 - 15.0 / 14.0, -8.0 / 7.0], rtol=0, atol=1e-14)
    # ESS = m n / (1 + 2 (rho_1 + rho_2)) with n = 3 (no odd-lag stop possible)
    assert od.ess(x) == pytest.approx(6.0 / (1.0 + 2.0 * (1.0 - 15.0 / 14.0 - 8.0 / 7.0)), rel=1e-14)
