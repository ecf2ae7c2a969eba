"""Config table for the five BASELINE.json workloads plus the BLR pin config.

Pinning follows SURVEY.md §8 "Config pinning" and the readings Q10-Q24 of
§8(c) (listed again in DESIGN.md §3).  Everything here is plain data.
"""
from __future__ import annotations

import json
import os
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


# --- the five BASELINE configs (SURVEY §5 "one JSON per BASELINE config") ---
# configs/cfg{1..5}.json hold every knob, with the readings of unstated fields listed under
# "assumed"; the generator in generate.py turns a config into a Problem.
CONFIG_DIR = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "configs")


def load_config(path_or_name: str) -> dict:
    """A config JSON (a path, or the name of one of configs/*.json) -> the generator's knobs."""
    path = path_or_name if path_or_name.endswith(".json") else os.path.join(CONFIG_DIR, path_or_name + ".json")
    with open(path) as f:
        d = json.load(f)
    a = d["arch"]
    arch = ArchSpec(a["kind"], tuple(NetSpec(tuple(n["widths"]), tuple(n["acts"]), tuple(bool(b) for b in n["bias"]))
                                     for n in a["nets"]), bool(a.get("has_b0", False)))
    act = d["active"]
    out = dict(cid=int(d["cid"]), arch=arch, noise=float(d["noise_sigma"]), prior=float(d["prior_sigma"]),
               active_frac=None if act == "all" else act.get("frac"), C=int(d["chains"]), L=int(d["L"]),
               eps=float(d["eps"]), S=int(d["S"]), mu=d["frozen_init"])
    if act != "all" and "count" in act:
        out["active_count"] = int(act["count"])
    out.update({k: int(v) for k, v in d["data"].items()})
    return out


CONFIGS = {name: load_config(name) for name in ("cfg1", "cfg2", "cfg3", "cfg4", "cfg5")}


def config_names():
    return list(CONFIGS.keys())
