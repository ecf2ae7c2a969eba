"""C-ABI contract tests that are not parity of the hot path itself: the dropped
normalising constant, the adapted step sizes surviving a fixed-eps call, the divergence flag,
setup validation (world, shards) and the binding's refusal of mistyped output buffers."""
import math

import numpy as np
import pytest

from hmcdata import ArchSpec, NetSpec, make_problem, make_tiny_problem
from oracle import hmc as ohmc

from gpu_util import gpu_grad, jittered_states, to_dev, torch_cuda

pytestmark = pytest.mark.gpu


def _abi():
    torch_cuda()
    from paper_2507_14652_b200 import abi
    return abi


@pytest.mark.parametrize("name", ["blr", "cfg2", "cfg4", "cfg4u"])
def test_logpost_const_matches_oracle(name):
    """hmc_logpost_const = -N log(sigma sqrt(2 pi)) - k log(sigma_p sqrt(2 pi)) (Q7)."""
    abi = _abi()
    prob = make_problem(name, n_chains=1)
    with abi.Context(prob) as c:
        got = abi.hmc_logpost_const(c.ctx)
    assert got == pytest.approx(ohmc.Target(prob).logpost_const(), rel=1e-14)


def test_normalised_logp_is_gaussian_density():
    """logp + const on the BLR pin config equals the log density of the Gaussian likelihood and
    prior written with the normal pdf itself: sum_n log N(y_n | F_n, sigma^2)
    + sum_{i in s} log N(theta_i | 0, sigma_p^2), F_n = x_n . w + b from the assembled parameters."""
    from scipy.stats import norm
    abi = _abi()
    prob = make_problem("blr", n_chains=2)
    th = jittered_states(prob, 2, scale=0.3)
    th[1] += 0.7
    with abi.Context(prob) as c:
        lp, _ = gpu_grad(c, th)
        const = abi.hmc_logpost_const(c.ctx)
    for ci in range(2):
        full = prob.frozen.astype(np.float64).copy()
        full[prob.idx] = th[ci]
        F = prob.x.astype(np.float64) @ full[:5] + full[5]
        want = (norm.logpdf(prob.y.astype(np.float64), loc=F, scale=prob.noise_sigma).sum()
                + norm.logpdf(th[ci].astype(np.float64), scale=prob.prior_sigma).sum())
        assert lp[ci] + const == pytest.approx(want, rel=1e-6)


def _state(prob, C):
    torch = torch_cuda()
    th = jittered_states(prob, C, scale=0.005)
    return th


def test_adapted_eps_survive_fixed_eps_call():
    """hmc_adapt's per-chain eps_bar stay in the context: a later call with eps > 0 must not
    overwrite them, so hmc_trajectory(eps = 0) after it runs at eps_bar (include/hmc.h:
    "the context keeps them").  Compared bitwise with a context that never ran the eps > 0 call."""
    abi = _abi()
    torch = torch_cuda()
    arch = ArchSpec("mlp", (NetSpec.plain((2, 24, 24, 1)),))
    prob = make_tiny_problem(arch, n=80, n_chains=3, seed=31, noise=0.2)
    th = jittered_states(prob, 3, scale=0.01)
    outs = []
    for detour in (False, True):
        with abi.Context(prob) as c:
            lp, g = gpu_grad(c, th)
            T, LP, G = to_dev(th, torch.float32), to_dev(lp, torch.float64), to_dev(g, torch.float32)
            eb = abi.hmc_adapt(c.ctx, T, LP, G, 1e-3, 6, 0, 12, 0.8)
            if detour:   # a fixed-eps trajectory on a scratch copy of the state
                T2, LP2, G2 = T.clone(), LP.clone(), G.clone()
                abi.hmc_trajectory(c.ctx, T2, LP2, G2, 3e-2, 6, 500)
            dH = torch.zeros(3, dtype=torch.float64, device="cuda")
            abi.hmc_trajectory(c.ctx, T, LP, G, 0.0, 6, 100, None, dH)
            torch.cuda.synchronize()
            outs.append((eb, T.cpu().numpy(), dH.cpu().numpy()))
    np.testing.assert_array_equal(outs[0][0], outs[1][0])
    np.testing.assert_array_equal(outs[0][1], outs[1][1])
    np.testing.assert_array_equal(outs[0][2], outs[1][2])


def test_divergence_counter():
    """hmc_divergences counts, per chain, the trajectories flagged by the oracle's definition
    (non-finite or |dH| > 1000) applied to the GPU's dH; a stable step flags none."""
    abi = _abi()
    torch = torch_cuda()
    arch = ArchSpec("mlp", (NetSpec.plain((1, 20, 20, 1)),))
    prob = make_tiny_problem(arch, n=64, n_chains=4, seed=32, noise=0.1)
    th = jittered_states(prob, 4, scale=0.01)
    S = 12
    with abi.Context(prob) as c:
        lp, g = gpu_grad(c, th)
        T, LP, G = to_dev(th, torch.float32), to_dev(lp, torch.float64), to_dev(g, torch.float32)
        dH = torch.empty(4, S, dtype=torch.float64, device="cuda")
        abi.hmc_sample(c.ctx, T, LP, G, 1e-4, 10, 0, S, None, None, dH)
        assert np.all(abi.hmc_divergences(c.ctx, reset=True) == 0)
        # a step size far beyond the stability limit: mostly divergent, energies up to inf / NaN
        for eps in (3e-2, 0.3):
            abi.hmc_sample(c.ctx, T, LP, G, eps, 10, 100, S, None, None, dH)
            d = dH.cpu().numpy()
            want = np.array([sum(ohmc.divergent(v) for v in d[ci]) for ci in range(4)], dtype=np.uint32)
            got = abi.hmc_divergences(c.ctx, reset=True)
            np.testing.assert_array_equal(got, want)
        assert want.sum() > 0
        assert np.all(abi.hmc_divergences(c.ctx) == 0)


def test_setup_validation_world_and_shards():
    """world must be 1, 2, 4 or 8; SINGLE mode needs world 1; DATA mode needs equal shards."""
    abi = _abi()
    prob = make_tiny_problem(ArchSpec("mlp", (NetSpec.plain((2, 5, 1)),)), n=8, seed=1)
    for kw in (dict(mode="chain", world=3, rank=0), dict(mode="chain", world=16, rank=1),
               dict(mode="single", world=2, rank=0), dict(mode="chain", world=2, rank=2)):
        with pytest.raises(abi.HmcError) as e:
            abi.Context(prob, **kw)
        assert e.value.code == abi.HMC_E_CONFIG, kw
    # DATA mode at world 1 with an n_global that is not world x the local rows
    with pytest.raises(abi.HmcError) as e:
        abi.Context(prob, mode="data", world=1, n_global=9)
    assert e.value.code == abi.HMC_E_CONFIG
    with abi.Context(prob, mode="chain", world=2, rank=1) as c:   # a valid chain-mode rank
        assert c.C == prob.n_chains


def test_binding_refuses_mistyped_outputs():
    """Output buffers of the wrong dtype, element count or layout raise before the call (the
    library would write C doubles into a float32 array, or into a temporary copy)."""
    abi = _abi()
    torch = torch_cuda()
    prob = make_tiny_problem(ArchSpec("mlp", (NetSpec.plain((2, 9, 1)),)), n=10, n_chains=2, seed=3)
    th = jittered_states(prob, 2)
    with abi.Context(prob) as c:
        lp, g = gpu_grad(c, th)
        with pytest.raises(TypeError):
            abi.hmc_grad(c.ctx, th, np.empty(2, dtype=np.float32), np.empty_like(g))
        with pytest.raises(TypeError):
            abi.hmc_grad(c.ctx, th, lp.copy(), np.empty(g.shape, dtype=np.float64))
        with pytest.raises(ValueError):
            abi.hmc_grad(c.ctx, th, np.empty(3, dtype=np.float64), np.empty_like(g))
        with pytest.raises(ValueError):   # non-contiguous in/out state
            big = np.zeros((2, 2 * prob.k), dtype=np.float32)
            abi.hmc_trajectory(c.ctx, big[:, ::2], lp.copy(), g.copy(), 1e-3, 2, 0)
        with pytest.raises(TypeError):   # torch output of the wrong dtype
            abi.hmc_grad(c.ctx, to_dev(th, torch.float32), torch.empty(2, device="cuda", dtype=torch.float32),
                         torch.empty(2, prob.k, device="cuda"))
        with pytest.raises(ValueError):
            abi.hmc_sample(c.ctx, th.copy(), lp.copy(), g.copy(), 1e-3, 2, 0, 3,
                           np.empty((2, 2, prob.k), dtype=np.float32))
