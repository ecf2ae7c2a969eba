"""GPU posterior predictive (hmc_predict, NEXT-4) against oracle.hmc.predictive on the same
samples: mean within 1e-6 relative (fp32 forward), variance within 1e-3 relative + a floor set by
the fp32 rounding of the outputs (var is a difference of fp64 moments of fp32 values)."""
import numpy as np
import pytest

from hmcdata import ArchSpec, NetSpec, make_problem, make_tiny_problem
from oracle import hmc as ohmc

from gpu_util import torch_cuda

pytestmark = pytest.mark.gpu

CASES = {
    "mlp_tc": (ArchSpec("mlp", (NetSpec.plain((2, 64, 96, 1)),)), dict(n=300, n_chains=4)),
    "mlp_ragged": (ArchSpec("mlp", (NetSpec.plain((3, 50, 30, 1)),)), dict(n=77, n_chains=3)),
    "deeponet": (ArchSpec("deeponet", (NetSpec.plain((5, 64, 64, 32)), NetSpec.plain((2, 64, 32), last="tanh")),
                          has_b0=True), dict(n_c=24, n_x=40, n_chains=4)),
}


@pytest.mark.parametrize("name", sorted(CASES))
def test_predict_matches_oracle(name):
    torch_cuda()
    from paper_2507_14652_b200 import abi
    arch, kw = CASES[name]
    prob = make_tiny_problem(arch, seed=31, active_frac=0.3, **kw)
    g = np.random.default_rng(5)
    S = 10   # not a multiple of n_chains: exercises the partial last batch
    base = prob.frozen[prob.idx].astype(np.float64)
    samples = (base[None, :] + 0.05 * g.normal(size=(S, prob.k))).astype(np.float32)
    with abi.Context(prob) as c:
        m, v = abi.hmc_predict(c, samples)
    mr, vr = ohmc.predictive(ohmc.Target(prob), samples.astype(np.float64))
    scale = np.abs(mr).max()
    np.testing.assert_allclose(m, mr, rtol=1e-5, atol=1e-6 * scale)
    np.testing.assert_allclose(v, vr, rtol=1e-3, atol=1e-6 * scale * scale)


def test_predict_cfg5_full_size_sampled():
    """cfg5 (1M pairs, 64 chains per batch) on 70 samples: checked on a subset of pairs."""
    torch_cuda()
    from paper_2507_14652_b200 import abi
    prob = make_problem("cfg5")
    g = np.random.default_rng(6)
    base = prob.frozen[prob.idx].astype(np.float64)
    samples = (base[None, :] + 0.01 * g.normal(size=(70, prob.k))).astype(np.float32)
    with abi.Context(prob) as c:
        m, v = abi.hmc_predict(c, samples)
    # oracle on 3 conditions x all points
    sub = make_problem("cfg5")
    sub.u = np.ascontiguousarray(prob.u[[0, 100, 511]])
    sub.v = np.ascontiguousarray(prob.v[[0, 100, 511]])
    mr, vr = ohmc.predictive(ohmc.Target(sub), samples.astype(np.float64))
    n_x = prob.q.shape[0]
    mg = np.concatenate([m[r * n_x:(r + 1) * n_x] for r in (0, 100, 511)])
    vg = np.concatenate([v[r * n_x:(r + 1) * n_x] for r in (0, 100, 511)])
    scale = np.abs(mr).max()
    np.testing.assert_allclose(mg, mr, rtol=1e-4, atol=1e-5 * scale)
    np.testing.assert_allclose(vg, vr, rtol=2e-2, atol=1e-5 * scale * scale)
