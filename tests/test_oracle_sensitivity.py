"""Pins of oracle/sensitivity.py (eqn:sensitivities P:193-197, eqn:threshold P:200-204) against
values fixed by hand computation, closed forms and finite differences of the forward pass."""
import os

import numpy as np
import pytest

from hmcdata import ArchSpec, NetSpec, make_tiny_problem
from oracle import network as onet
from oracle import sensitivity as osens

GOLD = os.path.join(os.path.dirname(__file__), "golden", "sensitivity_linear.txt")


def _golden():
    out = {}
    for line in open(GOLD):
        if line.startswith("#") or not line.strip():
            continue
        k, *v = line.split()
        out[k] = np.array([float(t) for t in v])
    return out


def _data(prob):
    if prob.arch.kind == "mlp":
        return {"x": prob.x, "y": prob.y}
    return {"u": prob.u, "q": prob.q, "v": prob.v}


def test_spec_worked_example_linear_net():
    """y = theta1 x + theta2 (an MLP with no hidden layer: W[1x1], b[1])."""
    g = _golden()
    arch = ArchSpec("mlp", (NetSpec.plain((1, 1)),))
    mu = np.array([0.7, -0.3])                    # any mean: the net is linear in theta
    S2 = osens.sensitivities(arch, mu, g["sigma"], {"x": g["x"][:, None]})
    np.testing.assert_allclose(S2, g["S2"], rtol=1e-14)


def test_zero_sigma_gives_zero_sensitivity():
    prob = make_tiny_problem(ArchSpec("mlp", (NetSpec.plain((2, 5, 1)),)), n=7, seed=1)
    sig = prob.sigma_vi.astype(np.float64).copy()
    sig[3] = 0.0
    S2 = osens.sensitivities(prob.arch, prob.frozen, sig, _data(prob))
    assert S2[3] == 0.0 and np.all(S2 >= 0)


def test_linear_in_theta_exact_variance():
    """Networks linear in theta: Eq. 16 is exact, Var[F(x)] = sum_i sigma_i^2 x_i^2 + sigma_b^2
    for F = w.x + b with independent Gaussian (w, b); averaged over data it equals sum S^2."""
    g = np.random.default_rng(3)
    d, n = 4, 9
    x = g.normal(size=(n, d))
    sig = g.uniform(0.01, 0.3, size=d + 1)
    arch = ArchSpec("mlp", (NetSpec.plain((d, 1)),))
    S2 = osens.sensitivities(arch, g.normal(size=d + 1), sig, {"x": x})
    var = (x * x) @ (sig[:d] ** 2) + sig[d] ** 2        # analytic Var[F(x_j)]
    assert S2.sum() == pytest.approx(var.mean(), rel=1e-13)


@pytest.mark.parametrize("kind", ["mlp", "mlp_sin", "deeponet"])
def test_definition_by_finite_differences(kind):
    """S_i^2 rebuilt from central differences of the FORWARD pass only (no reverse mode)."""
    if kind == "mlp":
        arch = ArchSpec("mlp", (NetSpec.plain((2, 4, 3, 1)),))
        prob = make_tiny_problem(arch, n=5, seed=2)
    elif kind == "mlp_sin":
        arch = ArchSpec("mlp", (NetSpec((1, 3, 1), ("sin", "identity"), (True, False)),))
        prob = make_tiny_problem(arch, n=6, seed=3)
    else:
        arch = ArchSpec("deeponet", (NetSpec.plain((3, 4, 2)), NetSpec.plain((2, 3, 2), last="tanh")),
                        has_b0=True)
        prob = make_tiny_problem(arch, n_c=3, n_x=4, seed=4)
    data = _data(prob)
    mu = prob.frozen.astype(np.float64)
    sig = prob.sigma_vi.astype(np.float64)
    S2 = osens.sensitivities(arch, mu, sig, data)
    h = 1e-6
    fd = np.zeros(mu.size)
    for i in range(mu.size):
        e = np.zeros(mu.size)
        e[i] = h
        dF = (onet.predict(arch, mu + e, data) - onet.predict(arch, mu - e, data)) / (2 * h)
        fd[i] = sig[i] ** 2 * np.mean(np.asarray(dF).ravel() ** 2)
    np.testing.assert_allclose(S2, fd, rtol=1e-6, atol=1e-12 * fd.max())


def test_scale_consistency():
    """Doubling every sigma quadruples every S^2 and leaves ranking and partition unchanged."""
    prob = make_tiny_problem(ArchSpec("mlp", (NetSpec.plain((2, 6, 1)),)), n=8, seed=5)
    data = _data(prob)
    S2 = osens.sensitivities(prob.arch, prob.frozen, prob.sigma_vi, data)
    S2b = osens.sensitivities(prob.arch, prob.frozen, 2.0 * prob.sigma_vi.astype(np.float64), data)
    np.testing.assert_allclose(S2b, 4.0 * S2, rtol=1e-14)
    np.testing.assert_array_equal(osens.ranking(S2), osens.ranking(S2b))
    for tau in (0.5, 0.9, 0.99):
        np.testing.assert_array_equal(osens.partition(S2, tau)[0], osens.partition(S2b, tau)[0])


def test_threshold_rules_and_ties():
    S2 = np.array([0.2, 0.5, 0.3])          # normalised scores {0.5, 0.3, 0.2}
    assert osens.n_hat(S2, 0.9) == 3        # c = 0.5, 0.8, 1.0: first c >= 0.9 is N = 3
    assert osens.n_hat(S2, 0.8) == 2
    assert osens.n_hat(S2, 0.9, rule="le") == 2   # eqn:threshold as printed: last c <= 0.9
    assert osens.n_hat(S2, 1.0) == 3              # tau = 1: every parameter (full HMC)
    act, fro = osens.partition(S2, 0.8)
    np.testing.assert_array_equal(act, [1, 2])
    np.testing.assert_array_equal(fro, [0])
    # ties ranked by ascending flat index
    np.testing.assert_array_equal(osens.ranking(np.array([1.0, 2.0, 1.0, 2.0])), [1, 3, 0, 2])
    # N^ nondecreasing in tau; partition respects the ranking
    g = np.random.default_rng(0).exponential(size=40)
    prev = 0
    for tau in np.linspace(0.05, 1.0, 20):
        n = osens.n_hat(g, tau)
        assert n >= prev
        prev = n
        a, f = osens.partition(g, tau)
        assert len(a) == n and len(a) + len(f) == 40
        if len(a) and len(f):
            assert g[a].min() >= g[f].max()
    c = osens.cumulative_fraction(g)
    assert np.all(np.diff(c) >= 0) and c[-1] == pytest.approx(1.0, rel=1e-14)
