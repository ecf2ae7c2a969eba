"""GPU split-R^ / ESS (hmc_diagnostics, NEXT-4) against oracle/diagnostics.py on the same draws,
and on draws from the GPU sampler itself (BLR)."""
import numpy as np
import pytest

from hmcdata import make_problem
from oracle import diagnostics as od

from gpu_util import gpu_grad, to_dev, torch_cuda

pytestmark = pytest.mark.gpu


def _ar1(g, C, S, k, phi):
    x = np.zeros((C, S, k))
    x[:, 0] = g.normal(size=(C, k)) / np.sqrt(1 - phi ** 2)
    for i in range(1, S):
        x[:, i] = phi * x[:, i - 1] + g.normal(size=(C, k))
    return x


@pytest.mark.parametrize("C,S,phi", [(4, 200, 0.0), (8, 501, 0.7), (3, 64, 0.95)])
def test_diagnostics_match_oracle(C, S, phi):
    torch_cuda()
    from paper_2507_14652_b200 import abi
    g = np.random.default_rng(C * 1000 + S)
    k = 37
    x = (_ar1(g, C, S, k, phi) + np.linspace(0, 1, k)[None, None, :]).astype(np.float32)
    x[:, :, 5] += np.arange(C)[:, None] * 3.0          # one unmixed parameter
    rh, es = abi.hmc_diagnostics(x)
    rr, er = od.diagnostics(x.astype(np.float64))
    np.testing.assert_allclose(rh, rr, rtol=1e-10)
    np.testing.assert_allclose(es, er, rtol=1e-9)
    assert rh[5] > 1.2


def test_diagnostics_of_gpu_samples_blr():
    torch = torch_cuda()
    from paper_2507_14652_b200 import abi
    prob = make_problem("blr", n_chains=4)
    with abi.Context(prob) as c:
        th = np.zeros((4, prob.k), dtype=np.float32)
        lp, g = gpu_grad(c, th)
        T, LP, G = to_dev(th, torch.float32), to_dev(lp, torch.float64), to_dev(g, torch.float32)
        from test_oracle_hmc import blr_closed_form, blr_eps
        A, mu = blr_closed_form(prob)
        eps = blr_eps(prob, A)
        S = 2000
        smp = torch.empty(4, S, prob.k, dtype=torch.float32, device="cuda")
        abi.hmc_sample(c.ctx, T, LP, G, eps, 4, 0, S, smp, None, None)
        torch.cuda.synchronize()
    x = smp[:, 200:, :].contiguous()
    rh, es = abi.hmc_diagnostics(x)            # device samples in, host results out
    rr, er = od.diagnostics(x.cpu().numpy().astype(np.float64))
    np.testing.assert_allclose(rh, rr, rtol=1e-9)
    np.testing.assert_allclose(es, er, rtol=1e-8)
    assert np.all(rh < 1.05) and np.all(es > 100)


def _every_lag_sum(rho):
    """The rule BDA3 does NOT use (stop after ANY lag t with rho_{t+1} + rho_{t+2} < 0); only to
    make sure the draws below separate it from the odd-lag rule."""
    s, n = 0.0, len(rho)
    for t in range(1, n):
        s += rho[t]
        if t + 2 < n and rho[t + 1] + rho[t + 2] < 0:
            break
    return s


def test_ess_odd_lag_truncation_on_gpu():
    """Short iid chains, whose autocorrelations flip sign at random lags: for many parameters the
    first negative pair follows an even lag, where the odd-lag rule (BDA3 11.8) and an every-lag
    rule give different ESS.  The GPU must follow the odd-lag rule (the oracle)."""
    torch_cuda()
    from paper_2507_14652_b200 import abi
    g = np.random.default_rng(77)
    C, S, k = 2, 24, 200
    x = g.normal(size=(C, S, k)).astype(np.float32)
    rh, es = abi.hmc_diagnostics(x)
    rr, er = od.diagnostics(x.astype(np.float64))
    np.testing.assert_allclose(es, er, rtol=1e-9)
    np.testing.assert_allclose(rh, rr, rtol=1e-10)
    differ = 0
    for j in range(k):
        ps = od.split_chains(x[:, :, j].astype(np.float64))
        rho = od.autocorr(ps)
        differ += int(abs(_every_lag_sum(rho) - od.truncated_sum(rho)) > 1e-12)
    assert differ >= 10, differ
