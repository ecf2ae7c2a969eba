"""Degenerate and boundary cases of the GPU path against the oracle (north_star tolerances):
a single active parameter (k = 1: a tensor-core weight, the DeepONet output bias b0), a single
datum / single pair, a mask confined to the narrow first layer, and a wide chain batch."""
import numpy as np
import pytest

from hmcdata import ArchSpec, NetSpec, make_tiny_problem
from oracle import hmc as ohmc

from gpu_util import assert_grad_close, gpu_grad, jittered_states, torch_cuda

pytestmark = pytest.mark.gpu

D = ArchSpec("deeponet", (NetSpec.plain((7, 130, 64, 50)), NetSpec.plain((3, 70, 50), last="tanh")), has_b0=True)
M = ArchSpec("mlp", (NetSpec.plain((3, 150, 70, 1)),))


def _ctx(prob):
    from paper_2507_14652_b200 import abi
    return abi.Context(prob)


def _check(prob, C, chains=None):
    th = jittered_states(prob, C)
    with _ctx(prob) as c:
        lp, g = gpu_grad(c, th)
    t = ohmc.Target(prob)
    for ci in (chains if chains is not None else range(C)):
        lr, gr = t.logp_grad(th[ci].astype(np.float64))
        assert_grad_close(lp[ci], g[ci], lr, gr, f"{prob.name} chain {ci}")


@pytest.mark.parametrize("which", ["tc_weight", "b0"])
def test_single_active_parameter(which):
    torch_cuda()
    prob = make_tiny_problem(D, n_c=40, n_x=37, n_chains=2, seed=61, noise=0.3)
    flat = prob.P - 1 if which == "b0" else 7 * 130 + 130 + 5  # b0 / a weight of the branch's 2nd layer
    prob.idx = np.array([flat], dtype=np.int32)
    _check(prob, 2)


def test_single_datum_and_single_pair():
    torch_cuda()
    _check(make_tiny_problem(M, n=1, n_chains=2, seed=62, noise=0.3, active_frac=0.5), 2)
    _check(make_tiny_problem(D, n_c=1, n_x=1, n_chains=2, seed=63, noise=0.3, active_frac=0.5), 2)


def test_mask_on_first_layer_only():
    torch_cuda()
    prob = make_tiny_problem(M, n=300, n_chains=2, seed=64, noise=0.3)
    prob.idx = np.arange(0, 3 * 150 + 150, 7, dtype=np.int32)   # first-layer weights and biases
    _check(prob, 2)


def test_wide_chain_batch():
    torch_cuda()
    _check(make_tiny_problem(M, n=97, n_chains=300, seed=65, noise=0.3, active_frac=0.3), 300, [0, 151, 299])


N = ArchSpec("mlp", (NetSpec.plain((1, 64, 64, 64, 64, 1)),))   # cfg2's widths: the narrow engine


def test_narrow_engine_edges():
    """The narrow engine on: a single datum (one 16-row block, 15 padding rows), a single active
    parameter (the output bias) and a first-layer-only mask, and a batch of 100 chains (more CTAs
    than the GPU holds at once: cluster waves instead of the grid mode)."""
    torch_cuda()
    from paper_2507_14652_b200 import abi
    p1 = make_tiny_problem(N, n=1, n_chains=2, seed=66, noise=0.3, active_frac=0.5)
    _check(p1, 2)
    p2 = make_tiny_problem(N, n=200, n_chains=2, seed=67, noise=0.3)
    p2.idx = np.array([p2.P - 1], dtype=np.int32)
    _check(p2, 2)
    p2.idx = np.arange(0, 64 + 64, 5, dtype=np.int32)                # layer-0 weights and biases
    _check(p2, 2)
    p3 = make_tiny_problem(N, n=1024, n_chains=100, seed=68, noise=0.3, active_frac=0.1)
    with abi.Context(p3) as c:
        assert abi.hmc_engine_info(c.ctx).startswith("narrow-simt (cluster"), abi.hmc_engine_info(c.ctx)
    _check(p3, 100, [0, 57, 99])
