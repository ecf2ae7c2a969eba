"""Parameter sensitivities and the tau-partition in fp64.  TEST
INFRASTRUCTURE ONLY (see oracle/__init__.py).

PAPER.md §3.1 "Sensitivity to network parameters":
  eqn:sensitivities   S_i^2 = sigma_i^2 / N_d * sum_j (dF_mu(x_j) / dtheta_i)^2
  eqn:threshold   N^ from the cumulative fraction of sum S^2, threshold tau
  §3.2                Theta_s = the N^ most sensitive parameters, the rest frozen
For operator networks the datum j is a (function u_c, query point y_x) pair ("or may be
replaced by the input function u_j for neural operators"): N_d = n_c * n_x and the
sum runs over all pairs.

The definition is followed literally: one reverse pass per datum of the network OUTPUT F
(not of the loss), the gradient squared and accumulated.  Slow (N_d reverse passes) and
obviously correct; used only at test sizes.

Reading of eqn:threshold ("tau rule"): the equation prints the LARGEST N with
cumulative fraction <= tau, while the surrounding text ("sufficient ... to capture 90 % of the
variance", §4.1.1) needs the SMALLEST N with fraction >= tau.  rule="ge" (default) implements
the text, rule="le" the equation as printed.  Ties in S^2 are ranked by ascending flat index.
"""
from __future__ import annotations

import numpy as np

from .network import layer_table, net_backward, net_forward


def output_grad_per_datum(arch, theta_full, data):
    """Yields (j, dF(x_j)/dtheta) over the flat parameters for every datum j (MLP: rows of x;
    DeepONet: pairs (c, x) in row-major order c * n_x + x)."""
    theta_full = np.asarray(theta_full, dtype=np.float64)
    P = theta_full.size
    if arch.kind == "mlp":
        x = np.asarray(data["x"], dtype=np.float64)
        for j in range(x.shape[0]):
            _, tape = net_forward(arch, theta_full, 0, x[j:j + 1])
            g = np.zeros(P)
            net_backward(arch, theta_full, 0, tape, np.ones((1, 1)), g)   # dF/dF = 1
            yield j, g
        return
    _, b0, _ = layer_table(arch)
    u = np.asarray(data["u"], dtype=np.float64)
    q = np.asarray(data["q"], dtype=np.float64)
    n_x = q.shape[1] if q.ndim == 3 else q.shape[0]   # unaligned: q [n_c, n_x, d_t]
    for c in range(u.shape[0]):
        B, tb = net_forward(arch, theta_full, 0, u[c:c + 1])
        for xi in range(n_x):
            qp = q[c, xi:xi + 1] if q.ndim == 3 else q[xi:xi + 1]
            T, tt = net_forward(arch, theta_full, 1, qp)
            g = np.zeros(P)
            # F = sum_k B_k T_k + b0: dF/dB_k = T_k, dF/dT_k = B_k, dF/db0 = 1
            net_backward(arch, theta_full, 0, tb, T, g)
            net_backward(arch, theta_full, 1, tt, B, g)
            if b0 is not None:
                g[b0] += 1.0
            yield c * n_x + xi, g


def sensitivities(arch, mu, sigma_vi, data):
    """S_i^2 = sigma_i^2 / N_d * sum_j (dF_mu(x_j)/dtheta_i)^2 (eqn:sensitivities),
    gradients evaluated at the VI mean mu."""
    mu = np.asarray(mu, dtype=np.float64)
    sq = np.zeros(mu.size)
    n_d = 0
    for _, g in output_grad_per_datum(arch, mu, data):
        sq += g * g
        n_d += 1
    s = np.asarray(sigma_vi, dtype=np.float64)
    return s * s * sq / n_d


def ranking(S2):
    """Parameters from most to least sensitive; equal S^2 by ascending flat index."""
    S2 = np.asarray(S2, dtype=np.float64)
    return np.lexsort((np.arange(S2.size), -S2))


def cumulative_fraction(S2):
    """c_n = sum_{i <= n} S^2_(rank i) / sum_j S^2_j, n = 1..N_Theta (eqn:threshold's ratio).
    The denominator is the same ranked running sum at n = N_Theta (left-to-right), so c_N_Theta = 1
    exactly and every c_n is one sequential sum over one division - a reading that fixes the
    rounding of the threshold decision ("tau rule")."""
    S2 = np.asarray(S2, dtype=np.float64)
    cs = np.cumsum(S2[ranking(S2)])
    tot = cs[-1] if cs.size else 0.0
    if tot <= 0:
        return np.zeros(S2.size)
    return cs / tot


def n_hat(S2, tau, rule="ge"):
    """N^ of eqn:threshold.  rule 'ge': min{N : c_N >= tau} (the text's reading);
    rule 'le': max{N_T : c_{N_T} <= tau} (the equation as printed)."""
    c = cumulative_fraction(S2)
    if c.size == 0 or c[-1] <= 0:
        return 0
    if rule == "le":
        ok = np.nonzero(c <= tau)[0]
        return int(ok[-1] + 1) if ok.size else 0
    # c is nondecreasing; compare with a relative slack for the fraction that equals tau exactly
    ok = np.nonzero(c >= tau * (1.0 - 1e-15))[0]
    return int(ok[0] + 1) if ok.size else int(c.size)


def partition(S2, tau, rule="ge"):
    """Theta_s (ascending flat indices of the N^ most sensitive parameters) and Theta_~s
    (§3.2)."""
    r = ranking(S2)
    n = n_hat(S2, tau, rule)
    active = np.sort(r[:n])
    frozen = np.sort(r[n:])
    return active.astype(np.int64), frozen.astype(np.int64)
