"""Pins of oracle.hmc.predictive (NEXT-4): a single sample reproduces the network's output with
zero variance; for a model linear in the sampled parameters the predictive mean is the model at
the sample mean and the variance is x^T Cov x (closed forms of a linear map of a sample)."""
import numpy as np
import pytest

from hmcdata import ArchSpec, NetSpec, make_problem, make_tiny_problem
from oracle import hmc as ohmc
from oracle import network as onet


def test_single_sample_is_the_network_output():
    prob = make_tiny_problem(ArchSpec("mlp", (NetSpec.plain((2, 5, 1)),)), n=9, seed=2, active_frac=0.5)
    t = ohmc.Target(prob)
    th = prob.frozen[prob.idx].astype(np.float64) + 0.1
    m, v = ohmc.predictive(t, th[None, :])
    np.testing.assert_allclose(m, onet.predict(prob.arch, t.assemble(th), t.data), rtol=1e-15)
    assert np.all(np.abs(v) <= 1e-15 * (1 + m * m))


def test_linear_model_mean_and_covariance():
    """BLR pin config: F = X w + b is linear in the active entries (w0, w2, w3, b)."""
    prob = make_problem("blr", n_chains=1)
    t = ohmc.Target(prob)
    g = np.random.default_rng(7)
    S = g.normal(size=(300, prob.k))
    m, v = ohmc.predictive(t, S)
    # F(theta_s) = F(0) + J theta_s with J the (constant) Jacobian wrt the active entries
    F0 = onet.predict(prob.arch, t.assemble(np.zeros(prob.k)), t.data)
    J = np.stack([onet.predict(prob.arch, t.assemble(np.eye(prob.k)[i]), t.data) - F0 for i in range(prob.k)], axis=1)
    mu_s = S.mean(axis=0)
    cov = (S - mu_s).T @ (S - mu_s) / S.shape[0]
    np.testing.assert_allclose(m, F0 + J @ mu_s, rtol=1e-12, atol=1e-12)
    np.testing.assert_allclose(v, np.einsum("ji,ik,jk->j", J, cov, J), rtol=1e-9, atol=1e-12)
