"""Config table for the five BASELINE.json workloads plus the BLR pin config.

Pinning follows SURVEY.md §8 "Config pinning" and the readings Q10-Q24 of
§8(c) (listed again in DESIGN.md §3).  Everything here is plain data.
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import Optional, Tuple

import numpy as np

ACTS = ("identity", "tanh", "sin")


@dataclass(frozen=True)
class NetSpec:
    """A feed-forward net: widths[0] inputs -> ... -> widths[-1] outputs.

    acts[l] / bias[l] describe linear layer l (0-based), l < len(widths)-1.
    PAPER.md P:68 (F_Theta), P:527-539 (Table 4, DeepONet nets are FFNNs).
    """

    widths: Tuple[int, ...]
    acts: Tuple[str, ...]
    bias: Tuple[bool, ...]

    def __post_init__(self):
        assert len(self.acts) == len(self.widths) - 1
        assert len(self.bias) == len(self.widths) - 1
        for a in self.acts:
            assert a in ACTS, a

    @staticmethod
    def plain(widths, hidden="tanh", last="identity"):
        n = len(widths) - 1
        acts = tuple([hidden] * (n - 1) + [last])
        return NetSpec(tuple(widths), acts, tuple([True] * n))


@dataclass(frozen=True)
class ArchSpec:
    """kind 'mlp' -> nets = (mlp,); kind 'deeponet' -> nets = (branch, trunk).

    DeepONet output = sum_k B_k(u) T_k(y) + b0.
    """

    kind: str
    nets: Tuple[NetSpec, ...]
    has_b0: bool = False


@dataclass
class Problem:
    """One seeded workload: architecture, data, frozen means, mask, HMC knobs.

    Arrays are float32 (the canonical inputs); idx is int32,
    strictly ascending.  For 'mlp': x [n, d_in], y [n].  For 'deeponet':
    u [n_c, m] (branch inputs), q [n_x, d_t] (trunk inputs; unaligned DeepONet: q [n_c, n_x, d_t],
    each pair its own query point), v [n_c, n_x].
    """

    name: str
    arch: ArchSpec
    frozen: np.ndarray
    idx: np.ndarray
    noise_sigma: float
    prior_sigma: float
    n_chains: int
    L: int
    eps: float
    S: int
    seed: int
    x: Optional[np.ndarray] = None
    y: Optional[np.ndarray] = None
    u: Optional[np.ndarray] = None
    q: Optional[np.ndarray] = None
    v: Optional[np.ndarray] = None
    inv_mass: Optional[np.ndarray] = None
    sigma_vi: Optional[np.ndarray] = None
    chain_ids: Optional[np.ndarray] = None
    meta: dict = field(default_factory=dict)

    @property
    def k(self) -> int:
        return int(self.idx.shape[0])

    @property
    def P(self) -> int:
        return int(self.frozen.shape[0])

    def initial_theta(self) -> np.ndarray:
        """theta_s(0) = mu_s for every chain."""
        return np.repeat(self.frozen[self.idx][None, :], self.n_chains, axis=0).astype(np.float32)


# --- the five BASELINE configs -------------------------------------------
# name -> dict of knobs; generator in generate.py turns these into a Problem.
CONFIGS = {
    "cfg1": dict(
        cid=1,
        arch=ArchSpec("mlp", (NetSpec.plain((1, 20, 20, 1)),)),
        n=64, noise=0.1, prior=1.0, active_frac=None, C=1, L=20, eps=1e-3, S=200,
        mu="n03",
    ),
    "cfg2": dict(
        cid=2,
        arch=ArchSpec("mlp", (NetSpec.plain((1, 64, 64, 64, 64, 1)),)),
        n=1024, noise=0.05, prior=1.0, active_frac=0.10, C=8, L=50, eps=5e-4, S=500,
        mu="n03",
    ),
    "cfg3": dict(
        cid=3,
        arch=ArchSpec("mlp", (NetSpec.plain((8, 256, 256, 256, 1)),)),
        n=16384, noise=0.05, prior=1.0, active_frac=0.05, C=32, L=100, eps=2e-4, S=200,
        mu="lecun",
    ),
    "cfg4": dict(
        cid=4,
        arch=ArchSpec(
            "deeponet",
            (
                NetSpec.plain((100, 128, 128, 128, 100), last="identity"),
                NetSpec.plain((1, 128, 128, 100), last="tanh"),
            ),
            has_b0=True,
        ),
        n_c=1000, n_x=100, noise=0.01, prior=1.0, active_frac=0.10, C=16, L=100, eps=1e-4,
        S=20, mu="lecun",
    ),
    "cfg5": dict(
        cid=5,
        arch=ArchSpec(
            "deeponet",
            (
                NetSpec.plain((5, 256, 256, 256, 256, 256), last="identity"),
                NetSpec.plain((2, 256, 256, 256, 256, 256), last="tanh"),
            ),
            has_b0=True,
        ),
        n_c=512, n_x=2048, noise=0.02, prior=1.0, active_count=20000, C=64, L=200,
        eps=5e-5, S=10, mu="lecun",
    ),
}


def config_names():
    return list(CONFIGS.keys())
