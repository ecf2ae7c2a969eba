"""GPU dual-averaging step-size adaptation (hmc_adapt, NEXT-2) against the fp64 oracle's
Algorithm-5 recursion on the same trajectories and Philox streams."""
import math

import numpy as np
import pytest

from hmcdata import make_problem
from oracle import hmc as ohmc

from gpu_util import to_dev, torch_cuda, gpu_grad

pytestmark = pytest.mark.gpu


def _run(prob, th, eps0, L, n, delta):
    torch = torch_cuda()
    from paper_2507_14652_b200 import abi
    with abi.Context(prob) as c:
        lp, g = gpu_grad(c, th)
        T, LP, G = to_dev(th, torch.float32), to_dev(lp, torch.float64), to_dev(g, torch.float32)
        C = th.shape[0]
        acc = torch.zeros(C, n, dtype=torch.uint8, device="cuda")
        dH = torch.zeros(C, n, dtype=torch.float64, device="cuda")
        eb = abi.hmc_adapt(c.ctx, T, LP, G, eps0, L, 0, n, delta, acc, dH)
        # sampling after adaptation with eps == 0 uses the per-chain eps_bar
        S = 50
        smp = torch.empty(C, S, prob.k, dtype=torch.float32, device="cuda")
        a2 = torch.empty(C, S, dtype=torch.uint8, device="cuda")
        d2 = torch.empty(C, S, dtype=torch.float64, device="cuda")
        abi.hmc_sample(c.ctx, T, LP, G, 0.0, L, n, S, smp, a2, d2)
        torch.cuda.synchronize()
        return eb, acc.cpu().numpy(), dH.cpu().numpy(), a2.cpu().numpy(), d2.cpu().numpy()


def test_adapt_cfg1_matches_oracle():
    """cfg1 (481 parameters, one chain): 60 adaptation trajectories, L = 20, eps0 = 1e-3,
    delta = 0.8.  (1) The GPU's dual-averaging recursion, replayed on the host (the oracle's
    da_update) from the GPU's own acceptance statistics min(1, exp(-dH)), gives the GPU's
    eps_bar to 1e-10 relative.  (2) The free-running chain makes the oracle's accept decisions
    until the step size grows to the point where fp32 / fp64 round-off can tip a decision near
    its margin: the first 12 decisions and dH agree."""
    prob = make_problem("cfg1")
    th0 = prob.frozen[prob.idx].astype(np.float32)[None, :]
    n = 60
    eb, acc, dH, _, _ = _run(prob, th0, 1e-3, prob.L, n, 0.8)
    st = ohmc.da_init(1e-3)
    for m in range(n):
        a = 0.0 if not np.isfinite(dH[0, m]) else min(1.0, math.exp(-dH[0, m]))
        st = ohmc.da_update(st, a, 0.8)
    assert eb[0] == pytest.approx(math.exp(st["log_epsbar"]), rel=1e-10)
    t = ohmc.Target(prob)
    eb_ref, eps_used, acc_ref, alph, _ = ohmc.adapt_chain(t, th0[0].astype(np.float64), 1e-3, prob.L, 0, 12, 0.8, 0)
    np.testing.assert_array_equal(acc[0, :12].astype(bool), acc_ref)
    d = dH[0, :12]
    a_gpu = np.where(np.isfinite(d), np.minimum(1.0, np.exp(-np.where(np.isfinite(d), d, 0.0))), 0.0)
    # |d alpha| <= alpha |d dH|: fp32 trajectories at the adapted (larger) steps differ from
    # fp64 by O(1e-3) in dH
    np.testing.assert_allclose(a_gpu, alph, rtol=0, atol=1e-2)


def test_adapt_blr_chains_hit_target_acceptance():
    """BLR pin config, 4 independent chains: after 1000 adaptation steps the 50 sampling
    trajectories at the per-chain eps_bar have mean acceptance statistic near 0.8."""
    prob = make_problem("blr", n_chains=4)
    th0 = np.zeros((4, prob.k), dtype=np.float32)
    eb, acc, dH, a2, d2 = _run(prob, th0, 0.5, 5, 1000, 0.8)
    assert np.all(np.isfinite(eb)) and np.all(eb > 0)
    alpha = np.minimum(1.0, np.exp(-d2))
    assert abs(alpha.mean() - 0.8) <= 0.1, (eb, alpha.mean())
    # per-chain steps are close to one another on the same posterior
    assert eb.max() / eb.min() < 1.5


def test_adapt_rejects_bad_arguments():
    torch = torch_cuda()
    from paper_2507_14652_b200 import abi
    prob = make_problem("blr", n_chains=1)
    with abi.Context(prob) as c:
        th = np.zeros((1, prob.k), dtype=np.float32)
        lp, g = gpu_grad(c, th)
        with pytest.raises(abi.HmcError):
            abi.hmc_adapt(c.ctx, th, lp, g, 0.1, 5, 0, 10, 1.5)
        with pytest.raises(abi.HmcError):      # eps == 0 before any adaptation
            abi.hmc_trajectory(c.ctx, th, lp, g, 0.0, 5, 0)
