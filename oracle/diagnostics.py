"""MCMC convergence diagnostics: split-R^ and effective
sample size, in fp64.  TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Definitions follow Gelman et al., Bayesian Data Analysis 3rd ed. §11.4-11.5, on SPLIT chains
(each of the C chains of S draws cut into two halves of n = floor(S / 2) draws; m = 2C):
  W = mean_j s_j^2 (within-chain variances, ddof 1),  B/n = var_j(mean_j) (ddof 1),
  var+ = (n - 1)/n W + B/n,   R^ = sqrt(var+ / W)                                     (11.3-11.4)
  V_t = 1/(m (n - t)) sum_j sum_{i > t} (psi_ij - psi_{i-t,j})^2   (variogram)
  rho_t = 1 - V_t / (2 var+)                                                           (11.7)
  ESS = m n / (1 + 2 sum_{t=1}^{T} rho_t), T the first odd lag with rho_{T+1} + rho_{T+2} < 0
                                                                                        (11.8)
"""
from __future__ import annotations

import numpy as np


def split_chains(x):
    """x [C, S] -> [2C, n] (the halves of every chain; a middle draw of odd S is dropped)."""
    x = np.asarray(x, dtype=np.float64)
    C, S = x.shape
    n = S // 2
    return np.concatenate([x[:, :n], x[:, S - n:]], axis=0)


def _moments(ps):
    m, n = ps.shape
    means = ps.mean(axis=1)
    W = ps.var(axis=1, ddof=1).mean()
    Bn = means.var(ddof=1)
    var_plus = (n - 1) / n * W + Bn
    return W, var_plus


def split_rhat(x):
    """x [C, S] draws of one scalar -> split-R^ (BDA3 11.4)."""
    W, var_plus = _moments(split_chains(x))
    return float(np.sqrt(var_plus / W))


def autocorr(ps):
    """rho_t, t = 0 .. n-1, of split chains ps [m, n] from the variogram (BDA3 11.7)."""
    m, n = ps.shape
    W, var_plus = _moments(ps)
    rho = [1.0]
    for t in range(1, n):
        V = np.sum((ps[:, t:] - ps[:, :-t]) ** 2) / (m * (n - t))
        rho.append(1.0 - V / (2.0 * var_plus))
    return np.array(rho)


def truncated_sum(rho):
    """sum_{t=1}^{T} rho_t with T the first ODD lag for which rho_{T+1} + rho_{T+2} < 0 (BDA3
    11.8: "the first odd positive integer T"); when no odd lag qualifies the sum runs to the
    last available lag n - 1.  Left-to-right order (the GPU kernel uses the same order)."""
    n = len(rho)
    s = 0.0
    t = 1
    while t < n:
        s += rho[t]                       # rho_T for the odd candidate T = t
        if t + 1 >= n:
            break
        if t + 2 < n and rho[t + 1] + rho[t + 2] < 0:
            break                         # T = t (odd)
        s += rho[t + 1]
        t += 2
    return s


def ess(x):
    """x [C, S] draws of one scalar -> effective sample size (BDA3 11.8)."""
    ps = split_chains(x)
    m, n = ps.shape
    return float(m * n / (1.0 + 2.0 * truncated_sum(autocorr(ps))))


def diagnostics(samples):
    """samples [C, S, k] -> (rhat [k], ess [k])."""
    samples = np.asarray(samples, dtype=np.float64)
    k = samples.shape[2]
    return (np.array([split_rhat(samples[:, :, j]) for j in range(k)]),
            np.array([ess(samples[:, :, j]) for j in range(k)]))
