"""Pins for oracle/hmc.py: leapfrog order, reversibility, closed-form BLR map and posterior,
Metropolis invariants (SURVEY §4 tier 1, §8(c) pins)."""
import math

import numpy as np
import pytest

from hmcdata import ArchSpec, NetSpec, make_problem, make_tiny_problem
from oracle import hmc as ohmc


def blr_closed_form(pr):
    """Gaussian conditional posterior of the BLR pin config: A = X_s^T X_s / s^2 + I/sp^2,
    mu = A^-1 X_s^T (y - X_~s mu_~s) / s^2.  Flat 0-4 = weights on x, flat 5 = bias."""
    X = np.hstack([pr.x.astype(np.float64), np.ones((pr.x.shape[0], 1))])
    y = pr.y.astype(np.float64)
    s = np.asarray(pr.idx)
    f = np.setdiff1d(np.arange(6), s)
    Xs, Xf = X[:, s], X[:, f]
    mu_f = pr.frozen.astype(np.float64)[f]
    A = Xs.T @ Xs / pr.noise_sigma ** 2 + np.eye(len(s)) / pr.prior_sigma ** 2
    mu = np.linalg.solve(A, Xs.T @ (y - Xf @ mu_f) / pr.noise_sigma ** 2)
    return A, mu


def blr_eps(pr, A):
    Minv = np.diag(pr.inv_mass.astype(np.float64))
    lam = np.max(np.real(np.linalg.eigvals(Minv @ A)))
    return 0.5 / math.sqrt(lam)


def test_blr_gradient_is_linear_closed_form():
    pr = make_problem("blr")
    A, mu = blr_closed_form(pr)
    t = ohmc.Target(pr)
    for th in (np.zeros(4), np.array([0.3, -1.0, 2.0, 0.5])):
        _, g = t.logp_grad(th)
        np.testing.assert_allclose(g, -A @ (th - mu), rtol=1e-9, atol=1e-8)


def test_blr_leapfrog_matches_exact_linear_map():
    """KDK on U = 1/2 (th-mu)^T A (th-mu): th~' = (I - e^2/2 M^-1 A) th~ + e M^-1 p,
    p' = p - e/2 A (th~ + th~') (SURVEY §8(c) leapfrog pin)."""
    pr = make_problem("blr")
    A, mu = blr_closed_form(pr)
    t = ohmc.Target(pr)
    eps = blr_eps(pr, A)
    Minv = np.diag(pr.inv_mass.astype(np.float64))
    g = np.random.default_rng(0)
    th0, p0 = mu + g.normal(size=4) * 0.01, g.normal(size=4)
    _, g0 = t.logp_grad(th0)
    L = 37
    th, p, _, _ = ohmc.leapfrog(t, th0, p0, g0, eps, L)
    tt, pp = th0 - mu, p0.copy()
    Mlin = np.eye(4) - 0.5 * eps * eps * Minv @ A
    for _ in range(L):
        tn = Mlin @ tt + eps * Minv @ pp
        pp = pp - 0.5 * eps * A @ (tt + tn)
        tt = tn
    np.testing.assert_allclose(th - mu, tt, rtol=0, atol=1e-10)
    np.testing.assert_allclose(p, pp, rtol=0, atol=1e-8 * np.max(np.abs(pp)))


def test_leapfrog_L0_identity_and_accept():
    pr = make_tiny_problem(ArchSpec("mlp", (NetSpec.plain((1, 5, 1)),)), n=10, seed=1)
    t = ohmc.Target(pr)
    th = pr.frozen[pr.idx].astype(np.float64)
    lp, g = t.logp_grad(th)
    p = np.ones(pr.k)
    a, b, _, c = ohmc.leapfrog(t, th, p, g, 0.1, 0)
    np.testing.assert_array_equal(a, th)
    np.testing.assert_array_equal(b, p)
    r = ohmc.trajectory(t, th, lp, g, 0.1, 0, 0, 0)
    assert r["accepted"] and r["dH"] == 0.0


def test_energy_error_is_second_order():
    """max |dH| over 100 trajectories at fixed T = L eps: halving eps divides it by ~4
    (ratio in [3.5, 4.5])."""
    pr = make_problem("blr")
    A, _ = blr_closed_form(pr)
    t = ohmc.Target(pr)
    eps0 = blr_eps(pr, A)
    g = np.random.default_rng(3)
    starts = [(g.normal(size=4) * 0.02 + 0.5, g.normal(size=4)) for _ in range(100)]
    maxes = []
    for m in (1, 2, 4):
        eps, L = eps0 / m, 10 * m
        worst = 0.0
        for th, pz in starts:
            p = pz / np.sqrt(pr.inv_mass)
            lp, gr = t.logp_grad(th)
            H0 = -lp + ohmc.kinetic(t, p)
            th1, p1, lp1, _ = ohmc.leapfrog(t, th, p, gr, eps, L)
            worst = max(worst, abs(-lp1 + ohmc.kinetic(t, p1) - H0))
        maxes.append(worst)
    r1, r2 = maxes[0] / maxes[1], maxes[1] / maxes[2]
    assert 3.5 <= r1 <= 4.5 and 3.5 <= r2 <= 4.5, (r1, r2)


def test_reversibility_nonlinear_net():
    """(th*, -p*) integrated back L steps recovers (th, -p) to 1e-10 in fp64."""
    pr = make_problem("cfg1")
    t = ohmc.Target(pr)
    th = pr.frozen[pr.idx].astype(np.float64)
    lp, g = t.logp_grad(th)
    p = ohmc.momentum(t, 0, 0)
    th1, p1, _, g1 = ohmc.leapfrog(t, th, p, g, pr.eps, pr.L)
    th2, p2, _, _ = ohmc.leapfrog(t, th1, -p1, g1, pr.eps, pr.L)
    assert np.max(np.abs(th2 - th)) <= 1e-10 * max(1.0, np.max(np.abs(th)))
    assert np.max(np.abs(p2 + p)) <= 1e-10 * max(1.0, np.max(np.abs(p)))


def test_blr_samples_recover_closed_form_posterior():
    """Sampler correctness: mean within 4 MCSE, covariance within 10 % of the closed-form
    Gaussian conditional (the frozen coordinates make it a conditional)."""
    pr = make_problem("blr", n_chains=4)
    A, mu = blr_closed_form(pr)
    Sigma = np.linalg.inv(A)
    t = ohmc.Target(pr)
    eps = blr_eps(pr, A)
    draws = []
    for c in range(4):
        s, acc, _ = ohmc.sample_chain(t, np.zeros(4), eps, 4, 0, 1600, c)
        assert acc.mean() > 0.8
        draws.append(s[100:])
    D = np.concatenate(draws)
    # batch-means MCSE
    nb = 30
    bm = np.array_split(D, nb)
    mcse = np.std([b.mean(axis=0) for b in bm], axis=0, ddof=1) / math.sqrt(nb)
    assert np.all(np.abs(D.mean(axis=0) - mu) < 4 * mcse + 1e-12), (D.mean(axis=0) - mu) / mcse
    C = np.cov(D.T)
    sd = np.sqrt(np.diag(Sigma))
    assert np.max(np.abs(C - Sigma) / np.outer(sd, sd)) < 0.10


def test_shift_invariance_of_decisions():
    """Adding a constant to log pi leaves every decision unchanged."""
    pr = make_tiny_problem(ArchSpec("mlp", (NetSpec.plain((1, 6, 1)),)), n=20, seed=2, noise=0.3)
    t = ohmc.Target(pr)

    class Shifted(ohmc.Target):
        def logp_grad(self, th):
            lp, g = super().logp_grad(th)
            return lp + 1234.5, g
    ts = Shifted(pr)
    th = pr.frozen[pr.idx].astype(np.float64)
    s1, a1, _ = ohmc.sample_chain(t, th, 0.05, 5, 0, 40, 0)
    s2, a2, _ = ohmc.sample_chain(ts, th, 0.05, 5, 0, 40, 0)
    assert 0 < a1.sum() < 40
    np.testing.assert_array_equal(a1, a2)


def test_tiny_step_accepts_everything():
    pr = make_tiny_problem(ArchSpec("mlp", (NetSpec.plain((1, 6, 1)),)), n=20, seed=3)
    t = ohmc.Target(pr)
    _, acc, dH = ohmc.sample_chain(t, pr.frozen[pr.idx], 1e-9, 3, 0, 50, 0)
    assert acc.all() and np.max(np.abs(dH)) < 1e-6


def test_nonfinite_proposal_rejected():
    pr = make_tiny_problem(ArchSpec("mlp", (NetSpec.plain((1, 4, 1)),)), n=8, seed=4)

    class Bad(ohmc.Target):
        calls = 0

        def logp_grad(self, th):
            Bad.calls += 1
            lp, g = super().logp_grad(th)
            return (lp if Bad.calls == 1 else float("nan")), g
    t = Bad(pr)
    th = pr.frozen[pr.idx].astype(np.float64)
    lp, g = t.logp_grad(th)
    r = ohmc.trajectory(t, th, lp, g, 0.01, 3, 0, 0)
    assert not r["accepted"]
    np.testing.assert_array_equal(r["theta"], th)


def test_divergence_flag_definition():
    """SPEC S:445 threshold as a flag (Q5): non-finite or |dH| > 1000."""
    assert ohmc.divergent(float("nan")) and ohmc.divergent(float("inf")) and ohmc.divergent(-float("inf"))
    assert ohmc.divergent(1000.5) and ohmc.divergent(-1e4)
    assert not ohmc.divergent(1000.0) and not ohmc.divergent(-999.0) and not ohmc.divergent(0.0)
