"""Seeded input generators (SURVEY.md §8(d) "Seeded generators", readings Q11-Q24).

rng(c, q) = np.random.default_rng(SeedSequence([c, q])) for config c and purpose q:
0 = inputs, 1 = noise, 2 = mu (frozen values), 3 = VI sigma, 4 = teacher / GRF /
coefficients, 5 = query points.  All arrays are returned as float32 (int32 for idx):
both the oracle (which upcasts to fp64) and the CUDA path start from bit-identical
values.  No HMC / posterior arithmetic lives here.
"""
from __future__ import annotations

import math
from typing import List, Optional, Tuple

import numpy as np

from .configs import CONFIGS, ArchSpec, NetSpec, Problem


def rng(c: int, q: int) -> np.random.Generator:
    return np.random.default_rng(np.random.SeedSequence([c, q]))


def layout_entries(arch: ArchSpec) -> List[Tuple[str, int, int, int]]:
    """(kind, offset, size, fan_in) in flat order: per net, per layer W[out x in]
    row-major then b[out]; DeepONet b0 last."""
    out = []
    off = 0
    for net in arch.nets:
        for l in range(len(net.widths) - 1):
            fi, fo = net.widths[l], net.widths[l + 1]
            out.append(("W", off, fo * fi, fi))
            off += fo * fi
            if net.bias[l]:
                out.append(("b", off, fo, fi))
                off += fo
    if arch.has_b0:
        out.append(("b0", off, 1, 1))
        off += 1
    return out


def n_params(arch: ArchSpec) -> int:
    e = layout_entries(arch)
    return e[-1][1] + e[-1][2] if e else 0


def frozen_values(arch: ArchSpec, mode: str, g: np.random.Generator) -> np.ndarray:
    """mu: 'n03' -> every entry ~ N(0, 0.3^2) (cfg1/cfg2 as stated);
    'lecun' -> W ~ N(0, 1/fan_in), biases and b0 = 0 (Q11)."""
    P = n_params(arch)
    if mode == "n03":
        return g.normal(0.0, 0.3, size=P).astype(np.float32)
    mu = np.zeros(P, dtype=np.float64)
    for kind, off, size, fan_in in layout_entries(arch):
        if kind == "W":
            mu[off:off + size] = g.normal(0.0, 1.0 / math.sqrt(fan_in), size=size)
    return mu.astype(np.float32)


def top_k_mask(sigma: np.ndarray, k: int) -> np.ndarray:
    """k largest sigma, ties by ascending flat index (Q13); returned ascending."""
    order = np.lexsort((np.arange(sigma.shape[0]), -sigma.astype(np.float64)))
    return np.sort(order[:k]).astype(np.int32)


def _grf_rbf(n_funcs: int, sensors: np.ndarray, length: float, g) -> np.ndarray:
    """Unit-variance RBF Gaussian random field at the sensors, sampled by eigh with
    eigenvalues clipped at 0 (Q19: Cholesky fails, min eigenvalue ~ -1e-14)."""
    d = sensors[:, None] - sensors[None, :]
    cov = np.exp(-(d * d) / (2.0 * length * length))
    w, V = np.linalg.eigh(cov)
    w = np.clip(w, 0.0, None)
    z = g.standard_normal((n_funcs, sensors.shape[0]))
    return (z * np.sqrt(w)[None, :]) @ V.T


def _antiderivative_pl(u: np.ndarray, s: np.ndarray, y: np.ndarray) -> np.ndarray:
    """Exact integral from 0 to y of the piecewise-linear interpolant of u (Q19)."""
    h = np.diff(s)
    seg = 0.5 * (u[:, 1:] + u[:, :-1]) * h[None, :]
    cum = np.concatenate([np.zeros((u.shape[0], 1)), np.cumsum(seg, axis=1)], axis=1)
    j = np.clip(np.searchsorted(s, y, side="right") - 1, 0, s.shape[0] - 2)
    t = y - s[j]
    slope = (u[:, j + 1] - u[:, j]) / h[j][None, :]
    return cum[:, j] + u[:, j] * t[None, :] + 0.5 * slope * (t * t)[None, :]


def _cone_field(c: np.ndarray, xs: np.ndarray, th: np.ndarray, g) -> np.ndarray:
    """Q18: p = sum_{m,q<4} x^q [(a_mq + b_mq.c) cos m th + (g_mq + e_mq.c) sin m th],
    coefficients scaled by 1/((1+m)(1+q)), normalised to unit std."""
    M = Q = 4
    alpha = g.standard_normal((M, Q))
    beta = g.standard_normal((M, Q, 5))
    gamma = g.standard_normal((M, Q))
    eta = g.standard_normal((M, Q, 5))
    out = np.zeros((c.shape[0], xs.shape[0]))
    for m in range(M):
        for q in range(Q):
            sc = 1.0 / ((1 + m) * (1 + q))
            a = (alpha[m, q] + c @ beta[m, q]) * sc
            b = (gamma[m, q] + c @ eta[m, q]) * sc
            out += (xs ** q)[None, :] * (a[:, None] * np.cos(m * th)[None, :]
                                         + b[:, None] * np.sin(m * th)[None, :])
    return out / out.std()


def _teacher(x: np.ndarray, g) -> np.ndarray:
    """cfg3 teacher MLP 8-32-32-1, tanh hidden, linear out, W ~ N(0,1/fan_in), b=0 (Q24)."""
    h = x.astype(np.float64)
    widths = (8, 32, 32, 1)
    for l in range(3):
        W = g.normal(0.0, 1.0 / math.sqrt(widths[l]), size=(widths[l + 1], widths[l]))
        h = h @ W.T
        if l < 2:
            h = np.tanh(h)
    return h[:, 0]


def make_problem(name: str, n_chains: Optional[int] = None) -> Problem:
    """Build one of cfg1..cfg5 or 'blr' exactly per SURVEY §8(d)."""
    if name == "blr":
        return make_blr_problem(n_chains or 4)
    # cfg4u: cfg4 with the query points drawn per function (unaligned DeepONet, NEXT-4, Q16)
    unaligned = name == "cfg4u"
    spec = CONFIGS["cfg4" if unaligned else name]
    cid = spec["cid"]
    arch: ArchSpec = spec["arch"]
    P = n_params(arch)
    mu = frozen_values(arch, spec["mu"], rng(cid, 2))
    sigma_vi = np.exp(rng(cid, 3).normal(-3.0, 1.0, size=P)).astype(np.float32)
    if spec.get("active_count"):
        k = spec["active_count"]
    elif spec["active_frac"] is None:
        k = P
    else:
        k = int(math.floor(spec["active_frac"] * P))
    idx = np.arange(P, dtype=np.int32) if k == P else top_k_mask(sigma_vi, k)
    C = n_chains or spec["C"]
    kw = dict(name=name, arch=arch, frozen=mu, idx=idx, noise_sigma=spec["noise"],
              prior_sigma=spec["prior"], n_chains=C, L=spec["L"], eps=spec["eps"],
              S=spec["S"], seed=cid - 1, sigma_vi=sigma_vi,
              chain_ids=np.arange(C, dtype=np.uint32))
    noise = spec["noise"]
    if name == "cfg1":
        x = rng(1, 0).uniform(-1.0, 1.0, size=spec["n"])
        y = np.sin(3.0 * x) + rng(1, 1).normal(0.0, noise, size=x.shape)
        return Problem(x=x[:, None].astype(np.float32), y=y.astype(np.float32), **kw)
    if name == "cfg2":
        x = rng(2, 0).uniform(-2.0, 2.0, size=spec["n"])
        y = x * np.sin(2.0 * x) + rng(2, 1).normal(0.0, noise, size=x.shape)
        return Problem(x=x[:, None].astype(np.float32), y=y.astype(np.float32), **kw)
    if name == "cfg3":
        x = rng(3, 0).normal(size=(spec["n"], 8))
        y = _teacher(x, rng(3, 4)) + rng(3, 1).normal(0.0, noise, size=spec["n"])
        return Problem(x=x.astype(np.float32), y=y.astype(np.float32), **kw)
    if unaligned:
        s = np.arange(100) / 99.0
        u = _grf_rbf(spec["n_c"], s, 0.2, rng(4, 4))
        yq = rng(4, 6).uniform(0.0, 1.0, size=(spec["n_c"], spec["n_x"]))
        G = np.stack([_antiderivative_pl(u[c:c + 1], s, yq[c])[0] for c in range(spec["n_c"])])
        v = G + rng(4, 1).normal(0.0, noise, size=(spec["n_c"], spec["n_x"]))
        return Problem(u=u.astype(np.float32), q=yq[:, :, None].astype(np.float32),
                       v=v.astype(np.float32), **kw)
    if name == "cfg4":
        s = np.arange(100) / 99.0
        u = _grf_rbf(spec["n_c"], s, 0.2, rng(4, 4))
        yq = rng(4, 5).uniform(0.0, 1.0, size=spec["n_x"])
        v = _antiderivative_pl(u, s, yq) + rng(4, 1).normal(0.0, noise, size=(spec["n_c"], spec["n_x"]))
        return Problem(u=u.astype(np.float32), q=yq[:, None].astype(np.float32),
                       v=v.astype(np.float32), **kw)
    if name == "cfg5":
        c = rng(5, 0).uniform(0.0, 1.0, size=(spec["n_c"], 5))
        xi = (np.arange(32) + 0.5) / 32.0
        thj = 2.0 * np.pi * np.arange(64) / 64.0
        xs = np.repeat(xi, 64)
        th = np.tile(thj, 32)
        v = _cone_field(c, xs, th, rng(5, 4)) + rng(5, 1).normal(0.0, noise, size=(spec["n_c"], 2048))
        q = np.stack([xs, th], axis=1)
        return Problem(u=c.astype(np.float32), q=q.astype(np.float32), v=v.astype(np.float32), **kw)
    raise KeyError(name)


def make_blr_problem(n_chains: int = 4) -> Problem:
    """Bayesian linear regression pin config ('BLR test config'):
    widths [5, 1], identity, P = 6, N = 200, idx {0,2,3,5}, flat 1 and 4 frozen at
    0.3 and -0.2, initial active values 0, inv_mass (1, 0.5, 2, 1), sigma 0.1, prior 1."""
    arch = ArchSpec("mlp", (NetSpec((5, 1), ("identity",), (True,)),))
    x = rng(0, 0).normal(size=(200, 5))
    wb = rng(0, 4).normal(size=6)
    y = x @ wb[:5] + wb[5] + rng(0, 1).normal(0.0, 0.1, size=200)
    frozen = np.array([0.0, 0.3, 0.0, 0.0, -0.2, 0.0], dtype=np.float32)
    return Problem(name="blr", arch=arch, frozen=frozen, idx=np.array([0, 2, 3, 5], dtype=np.int32),
                   noise_sigma=0.1, prior_sigma=1.0, n_chains=n_chains, L=20, eps=0.0, S=10000,
                   seed=0, x=x.astype(np.float32), y=y.astype(np.float32),
                   inv_mass=np.array([1.0, 0.5, 2.0, 1.0], dtype=np.float32),
                   chain_ids=np.arange(n_chains, dtype=np.uint32), meta={"w_true": wb})


def make_tiny_problem(arch: ArchSpec, *, n: int = 0, n_c: int = 0, n_x: int = 0,
                      active_frac: float = 1.0, n_chains: int = 1, seed: int = 0,
                      noise: float = 0.1, prior: float = 1.0, mu_scale: float = 0.5,
                      inv_mass: bool = False, L: int = 10, eps: float = 1e-3,
                      unaligned: bool = False) -> Problem:
    """Small seeded problems for pins and parity tests (any arch, ragged sizes)."""
    g = np.random.default_rng(np.random.SeedSequence([1000 + seed, 0]))
    P = n_params(arch)
    mu = g.normal(0.0, mu_scale, size=P).astype(np.float32)
    sigma_vi = np.exp(g.normal(-3.0, 1.0, size=P)).astype(np.float32)
    k = max(1, int(math.floor(active_frac * P)))
    idx = np.arange(P, dtype=np.int32) if k == P else top_k_mask(sigma_vi, k)
    im = g.uniform(0.5, 2.0, size=k).astype(np.float32) if inv_mass else None
    kw = dict(name=f"tiny{seed}", arch=arch, frozen=mu, idx=idx, noise_sigma=noise,
              prior_sigma=prior, n_chains=n_chains, L=L, eps=eps, S=1, seed=seed,
              sigma_vi=sigma_vi, inv_mass=im, chain_ids=np.arange(n_chains, dtype=np.uint32))
    if arch.kind == "mlp":
        d = arch.nets[0].widths[0]
        x = g.normal(size=(n, d)).astype(np.float32)
        y = g.normal(size=n).astype(np.float32)
        return Problem(x=x, y=y, **kw)
    m = arch.nets[0].widths[0]
    dt = arch.nets[1].widths[0]
    u = g.normal(size=(n_c, m)).astype(np.float32)
    q = g.uniform(0.0, 1.0, size=((n_c, n_x, dt) if unaligned else (n_x, dt))).astype(np.float32)
    v = g.normal(size=(n_c, n_x)).astype(np.float32)
    return Problem(u=u, q=q, v=v, **kw)
