"""Reduced-space HMC (Algorithm 2) in fp64.  TEST INFRASTRUCTURE ONLY (oracle/__init__.py).

Target: P(Theta_s | D, mu_~s) with Theta_~s fixed at mu_~s and prior
P(Theta_s | Theta_~s) = independent N(0, sigma_p^2) on the active coordinates only
(Q8).  U = -log[P(D|Theta)P(Theta)] + Z, constants dropped (Q7).
K = 1/2 p^T M^-1 p (P:110-114 read as the Gaussian log-density, Q1), M diagonal (Q6).
Leapfrog in kick-drift-kick form with the start gradient cached (Q2).
MH (Algorithm 1/2): accept iff r > u <=> ln u < H0 - H* strictly,
non-finite H* rejects (Q4, Q5).  No momentum negation (Q3).
"""
from __future__ import annotations

import math

import numpy as np

from . import network, philox


class Target:
    """Reduced log-posterior over the active coordinates idx."""

    def __init__(self, problem):
        self.arch = problem.arch
        self.frozen = np.asarray(problem.frozen, dtype=np.float64)
        self.idx = np.asarray(problem.idx, dtype=np.int64)
        self.sigma = float(problem.noise_sigma)
        self.sigma_p = float(problem.prior_sigma)
        k = self.idx.shape[0]
        self.inv_mass = (np.ones(k) if problem.inv_mass is None
                         else np.asarray(problem.inv_mass, dtype=np.float64))
        if problem.arch.kind == "mlp":
            self.data = {"x": np.asarray(problem.x, dtype=np.float64),
                         "y": np.asarray(problem.y, dtype=np.float64)}
        else:
            self.data = {"u": np.asarray(problem.u, dtype=np.float64),
                         "q": np.asarray(problem.q, dtype=np.float64),
                         "v": np.asarray(problem.v, dtype=np.float64)}
        self.seed = int(problem.seed)

    def assemble(self, theta_s):
        """Theta = mu with Theta[idx] = theta_s."""
        full = self.frozen.copy()
        full[self.idx] = np.asarray(theta_s, dtype=np.float64)
        return full

    def logp_grad(self, theta_s):
        """log P(D|Theta_s, mu_~s) + log P(Theta_s) without constants, and its gradient over
        the active coordinates (ascent direction)."""
        th = np.asarray(theta_s, dtype=np.float64)
        ll, g_full, _ = network.loglik_grad(self.arch, self.assemble(th), self.data, self.sigma)
        sp2 = self.sigma_p ** 2
        lp = ll - np.dot(th, th) / (2.0 * sp2)
        g = g_full[self.idx] - th / sp2
        return lp, g

    def grad_scale(self, theta_s, kappa=0.0):
        """Element-wise summation scale S_i for gradient tolerances (Q26; kappa: Q26b, see
        network.grad_abs_scale)."""
        th = np.asarray(theta_s, dtype=np.float64)
        S = network.grad_abs_scale(self.arch, self.assemble(th), self.data, self.sigma, kappa)
        return S[self.idx] + np.abs(th) / self.sigma_p ** 2

    def logpost_const(self):
        """Dropped normalising constant -N log(sigma sqrt(2 pi)) - k log(sigma_p sqrt(2 pi))."""
        if self.arch.kind == "mlp":
            n = self.data["y"].shape[0]
        else:
            n = self.data["v"].size
        k = self.idx.shape[0]
        return (-n * math.log(self.sigma * math.sqrt(2 * math.pi))
                - k * math.log(self.sigma_p * math.sqrt(2 * math.pi)))


def momentum(target, it, chain):
    """p ~ N(0, M): p_j = sqrt(m_j) z_j, z from Philox tag 0."""
    z = philox.normals(target.seed, 0, it, chain, target.idx.shape[0])
    return np.sqrt(1.0 / target.inv_mass) * z


def kinetic(target, p):
    return 0.5 * np.dot(p * target.inv_mass, p)


def leapfrog(target, theta, p, grad, eps, L):
    """T_s of P:126 in KDK form: p += eps/2 g; L times {theta += eps M^-1 p; g = grad(theta);
    p += eps g (eps/2 on the last)}.  Returns (theta, p, logp, grad); L = 0 is the identity
    (logp None then)."""
    theta = np.asarray(theta, dtype=np.float64).copy()
    p = np.asarray(p, dtype=np.float64).copy()
    g = np.asarray(grad, dtype=np.float64).copy()
    lp = None
    if L == 0:
        return theta, p, lp, g
    p = p + 0.5 * eps * g
    for step in range(L):
        theta = theta + eps * target.inv_mass * p
        lp, g = target.logp_grad(theta)
        p = p + (0.5 * eps if step == L - 1 else eps) * g
    return theta, p, lp, g


def trajectory(target, theta, logp, grad, eps, L, it, chain):
    """One Algorithm-2 iteration.  Returns dict with the new state, the accept
    flag, dH = H* - H0 and the proposal (theta*, p*)."""
    p0 = momentum(target, it, chain)
    H0 = -float(logp) + kinetic(target, p0)
    th1, p1, lp1, g1 = leapfrog(target, theta, p0, grad, eps, L)
    if L == 0:
        lp1 = float(logp)
    H1 = -float(lp1) + kinetic(target, p1)
    u = philox.mh_uniform(target.seed, it, chain)
    dH = H1 - H0
    accept = bool(np.isfinite(H1) and math.log(u) < H0 - H1)
    if accept:
        new = (th1, float(lp1), g1)
    else:
        new = (np.asarray(theta, dtype=np.float64), float(logp), np.asarray(grad, dtype=np.float64))
    return {"theta": new[0], "logp": new[1], "grad": new[2], "accepted": accept, "dH": dH,
            "theta_prop": th1, "p_prop": p1, "p0": p0, "H0": H0, "H1": H1, "u": u}


# Divergence diagnostic ("gradient explosion"; SPEC S:445's |dH| > 1000
# threshold, read as a flag only - Q5 keeps the exact Metropolis test as the sole decision).
DIVERGENCE_DH = 1000.0


def divergent(dH):
    """A trajectory is divergent when its energy error is non-finite or |dH| > 1000."""
    return bool(not math.isfinite(dH) or abs(dH) > DIVERGENCE_DH)


def sample_chain(target, theta0, eps, L, iter0, S, chain):
    """S consecutive trajectories for one chain (P:234 while-loop); burn-in is the caller's."""
    theta = np.asarray(theta0, dtype=np.float64)
    lp, g = target.logp_grad(theta)
    k = theta.shape[0]
    samples = np.empty((S, k))
    acc = np.zeros(S, dtype=bool)
    dHs = np.empty(S)
    for s in range(S):
        r = trajectory(target, theta, lp, g, eps, L, iter0 + s, chain)
        theta, lp, g = r["theta"], r["logp"], r["grad"]
        samples[s] = theta
        acc[s] = r["accepted"]
        dHs[s] = r["dH"]
    return samples, acc, dHs


# ---- step-size adaptation ----
# "the step size is computed using the step size adaptation method proposed in
# Algorithm 5 of [Hoffman & Gelman]" with the acceptance rate fixed at 80 %.  Dual averaging:
#   mu = log(10 eps0), Hbar_0 = 0, log epsbar_0 = 0, gamma = 0.05, t0 = 10, kappa = 0.75;
#   after adaptation trajectory m (run with eps_{m-1}) with acceptance statistic
#   alpha_m = min(1, exp(H0 - H*)) (0 for a non-finite H*):
#     Hbar_m = (1 - 1/(m + t0)) Hbar_{m-1} + (delta - alpha_m) / (m + t0)
#     log eps_m = mu - sqrt(m) / gamma * Hbar_m
#     log epsbar_m = m^-kappa log eps_m + (1 - m^-kappa) log epsbar_{m-1}
#   and sampling after adaptation uses epsbar_M.
DA_GAMMA, DA_T0, DA_KAPPA = 0.05, 10.0, 0.75


def accept_stat(H0, H1):
    """alpha = min(1, exp(H0 - H*)), 0 when H* is not finite (the proposal is rejected)."""
    if not np.isfinite(H1):
        return 0.0
    d = H0 - H1
    return 1.0 if d >= 0 else math.exp(d)


def da_init(eps0):
    return {"mu": math.log(10.0 * eps0), "hbar": 0.0, "log_epsbar": 0.0, "m": 0, "log_eps": math.log(eps0)}


def da_update(st, alpha, delta):
    """One dual-averaging step (Algorithm 5 of Hoffman & Gelman, quoted above)."""
    m = st["m"] + 1
    eta = 1.0 / (m + DA_T0)
    hbar = (1.0 - eta) * st["hbar"] + eta * (delta - alpha)
    log_eps = st["mu"] - math.sqrt(m) / DA_GAMMA * hbar
    w = m ** (-DA_KAPPA)
    log_epsbar = w * log_eps + (1.0 - w) * st["log_epsbar"]
    return {"mu": st["mu"], "hbar": hbar, "log_epsbar": log_epsbar, "m": m, "log_eps": log_eps}


def adapt_chain(target, theta0, eps0, L, iter0, n_adapt, delta, chain):
    """n_adapt adaptation trajectories of one chain (warm-up; the state advances as in
    sampling).  Returns (epsbar, per-trajectory eps used, accept flags, alphas, final state)."""
    theta = np.asarray(theta0, dtype=np.float64)
    lp, g = target.logp_grad(theta)
    st = da_init(eps0)
    eps_used, accs, alphas = [], [], []
    for s in range(n_adapt):
        eps = math.exp(st["log_eps"])
        r = trajectory(target, theta, lp, g, eps, L, iter0 + s, chain)
        theta, lp, g = r["theta"], r["logp"], r["grad"]
        a = accept_stat(r["H0"], r["H1"])
        st = da_update(st, a, delta)
        eps_used.append(eps)
        accs.append(r["accepted"])
        alphas.append(a)
    return math.exp(st["log_epsbar"]), np.array(eps_used), np.array(accs), np.array(alphas), (theta, lp, g)


# ---- posterior predictive ----
def predictive(target, samples):
    """Mean and (population) variance over the samples of F(x_j) for every datum j
    (P:401 / P:480: predictions reported as mean +- 3 sd over the HMC samples).  The frozen
    parameters stay at mu; MLP -> [n], DeepONet -> [n_c * n_x] row-major."""
    vals = []
    for th in np.asarray(samples, dtype=np.float64):
        F = network.predict(target.arch, target.assemble(th), target.data)
        vals.append(np.asarray(F, dtype=np.float64).ravel())
    V = np.array(vals)
    m = V.mean(axis=0)
    return m, (V * V).mean(axis=0) - m * m
