"""Pins of the dual-averaging step-size adaptation (oracle/hmc.py; P:490,
Algorithm 5 of Hoffman & Gelman): closed forms of the recursion, the target acceptance on a
Gaussian posterior, monotonicity in delta."""
import math

import numpy as np
import pytest

from hmcdata import make_problem
from oracle import hmc as ohmc


def test_recursion_fixed_point_at_target_acceptance():
    """alpha_m = delta for every m: Hbar = 0, log eps_m = mu, and since 1^-kappa = 1 the average
    log epsbar_m = mu from m = 1 on: epsbar = 10 eps0 exactly."""
    st = ohmc.da_init(0.02)
    for _ in range(25):
        st = ohmc.da_update(st, 0.8, 0.8)
        assert st["hbar"] == 0.0
        assert st["log_eps"] == pytest.approx(math.log(0.2), rel=1e-15)
        assert st["log_epsbar"] == pytest.approx(math.log(0.2), rel=1e-15)


def test_recursion_first_two_steps_by_hand():
    eps0, delta = 0.1, 0.8
    mu = math.log(1.0)
    st = ohmc.da_update(ohmc.da_init(eps0), 0.0, delta)
    h1 = 0.8 / 11.0
    assert st["hbar"] == pytest.approx(h1, rel=1e-15)
    assert st["log_eps"] == pytest.approx(mu - h1 / 0.05, rel=1e-14)
    assert st["log_epsbar"] == pytest.approx(mu - h1 / 0.05, rel=1e-14)   # 1^-kappa = 1
    st = ohmc.da_update(st, 1.0, delta)
    h2 = (1 - 1 / 12.0) * h1 + (0.8 - 1.0) / 12.0
    le2 = mu - math.sqrt(2) / 0.05 * h2
    w = 2 ** -0.75
    assert st["hbar"] == pytest.approx(h2, rel=1e-14)
    assert st["log_eps"] == pytest.approx(le2, rel=1e-14)
    assert st["log_epsbar"] == pytest.approx(w * le2 + (1 - w) * (mu - h1 / 0.05), rel=1e-14)


def test_accept_stat():
    assert ohmc.accept_stat(1.0, 0.5) == 1.0
    assert ohmc.accept_stat(1.0, 1.5) == pytest.approx(math.exp(-0.5))
    assert ohmc.accept_stat(1.0, float("nan")) == 0.0
    assert ohmc.accept_stat(1.0, float("inf")) == 0.0


def _probe(t, theta, eps, L, it0, n):
    lp, g = t.logp_grad(theta)
    acc = []
    for s in range(n):
        r = ohmc.trajectory(t, theta, lp, g, eps, L, it0 + s, 0)
        theta, lp, g = r["theta"], r["logp"], r["grad"]
        acc.append(ohmc.accept_stat(r["H0"], r["H1"]))
    return float(np.mean(acc))


def test_adapted_step_hits_target_acceptance_on_gaussian_posterior():
    """BLR pin config (Gaussian posterior): delta = 0.8 -> mean acceptance statistic of a
    500-trajectory probe at epsbar within 0.8 +- 0.07, after 1000 adaptation steps
    (the averaged epsbar lags the iterates and needs the longer warm-up)."""
    prob = make_problem("blr", n_chains=1)
    t = ohmc.Target(prob)
    theta0 = np.zeros(prob.k)
    eps_bar, eps_used, acc, alph, (th, _, _) = ohmc.adapt_chain(t, theta0, 0.5, 5, 0, 1000, 0.8, 0)
    a = _probe(t, th, eps_bar, 5, 10_000, 500)
    assert abs(a - 0.8) <= 0.07, (eps_bar, a)


def test_higher_target_gives_smaller_step():
    prob = make_problem("blr", n_chains=1)
    t = ohmc.Target(prob)
    e_hi = ohmc.adapt_chain(t, np.zeros(prob.k), 0.5, 5, 0, 300, 0.95, 0)[0]
    e_lo = ohmc.adapt_chain(t, np.zeros(prob.k), 0.5, 5, 0, 300, 0.6, 0)[0]
    assert e_hi < e_lo
