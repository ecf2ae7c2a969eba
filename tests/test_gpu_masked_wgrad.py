"""Masked weight gradient (csrc/masked_wgrad.cuh: the mask's entries only, P:257 last sentence)
forced on every hidden layer it takes (hmc_debug_set_engine(4)), against the fp64 oracle under
the north_star tolerances, and against the dense weight-gradient engines on the same inputs.
Shapes cover ragged row counts (rows not a multiple of the 16-row stage), row segments, several
task blocks (dense masks: more than 512 tasks), bias-only rows and both net kinds."""
import numpy as np
import pytest

from hmcdata import ArchSpec, NetSpec, make_problem, make_tiny_problem
from oracle import hmc as ohmc
from oracle import sensitivity as osens

from gpu_util import assert_grad_close, gpu_grad, jittered_states, torch_cuda

pytestmark = pytest.mark.gpu


def _ctx(prob):
    torch_cuda()
    from paper_2507_14652_b200 import abi
    return abi.Context(prob)


class _Mode:
    def __init__(self, mode):
        self.mode = mode

    def __enter__(self):
        from paper_2507_14652_b200 import abi
        abi.hmc_debug_set_engine(self.mode)

    def __exit__(self, *a):
        from paper_2507_14652_b200 import abi
        abi.hmc_debug_set_engine(0)


CASES = {
    # ragged rows (333), 36 -> 44 -> 40 hidden layers, 30 % of the parameters
    "mlp": (ArchSpec("mlp", (NetSpec.plain((3, 36, 44, 40, 1)),)), dict(n=333, active_frac=0.3), 31),
    # sparse mask (3 %): many rows with a bias-only or single-entry task
    "mlp_sparse": (ArchSpec("mlp", (NetSpec.plain((2, 64, 64, 1)),)), dict(n=517, active_frac=0.03), 32),
    # dense 128 x 128 layer: 2064 tasks -> several task blocks of 512 lanes
    "mlp_dense": (ArchSpec("mlp", (NetSpec.plain((1, 128, 128, 1)),)), dict(n=200, active_frac=1.0), 33),
    # DeepONet, ragged conditions / points, 100-wide input layer (n_in = 100)
    "deeponet": (ArchSpec("deeponet", (NetSpec.plain((100, 40, 32)), NetSpec.plain((2, 24, 32), last="tanh")),
                          has_b0=True), dict(n_c=45, n_x=77, active_frac=0.25), 34),
}


@pytest.mark.parametrize("name", sorted(CASES))
def test_masked_wgrad_tiny(name):
    from paper_2507_14652_b200 import abi
    arch, kw, seed = CASES[name]
    prob = make_tiny_problem(arch, n_chains=3, seed=seed, noise=0.3, **kw)
    th = jittered_states(prob, 3)
    with _Mode(4):
        with _ctx(prob) as c:
            assert "masked wgrad" in abi.hmc_engine_info(c.ctx), abi.hmc_engine_info(c.ctx)
            lp, g = gpu_grad(c, th)
    with _Mode(2):  # the dense per-layer engines on the same inputs
        with _ctx(prob) as c:
            assert "masked wgrad" not in abi.hmc_engine_info(c.ctx)
            lp_d, g_d = gpu_grad(c, th)
    t = ohmc.Target(prob)
    for ci in range(3):
        lr, gr = t.logp_grad(th[ci].astype(np.float64))
        assert_grad_close(lp[ci], g[ci], lr, gr, f"{name} masked chain {ci}")
        assert_grad_close(lp_d[ci], g_d[ci], lr, gr, f"{name} dense chain {ci}")
    # same likelihood pass: log pi identical; gradients differ only by summation order
    np.testing.assert_array_equal(lp, lp_d)


@pytest.mark.parametrize("cfg,C", [("cfg4", 2), ("cfg5", 4), ("cfg3", 2)])
def test_masked_wgrad_full_size(cfg, C):
    """Full-size problems (row segments, k-slot compaction of 8.8k / 20k / 6.7k entries)."""
    from paper_2507_14652_b200 import abi
    prob = make_problem(cfg, n_chains=C)
    th = jittered_states(prob, C)
    with _Mode(4):
        with _ctx(prob) as c:
            assert "masked wgrad" in abi.hmc_engine_info(c.ctx)
            lp, g = gpu_grad(c, th)
    t = ohmc.Target(prob)
    for ci in (0, C - 1):
        lr, gr = t.logp_grad(th[ci].astype(np.float64))
        assert_grad_close(lp[ci], g[ci], lr, gr, f"{cfg} chain {ci}")


def test_masked_wgrad_trajectory_decisions():
    """A 10-step trajectory on the masked path: end states within 1e-4 and the oracle's decision."""
    import torch
    from paper_2507_14652_b200 import abi
    arch, kw, seed = CASES["mlp"]
    prob = make_tiny_problem(arch, n_chains=2, seed=seed, noise=0.3, **kw)
    th = jittered_states(prob, 2)
    t = ohmc.Target(prob)
    with _Mode(4):
        with _ctx(prob) as c:
            T = torch.as_tensor(th, device="cuda").contiguous()
            LP = torch.empty(2, dtype=torch.float64, device="cuda")
            G = torch.empty(2, prob.k, dtype=torch.float32, device="cuda")
            abi.hmc_grad(c.ctx, T, LP, G)
            acc = torch.zeros(2, dtype=torch.uint8, device="cuda")
            abi.hmc_trajectory(c.ctx, T, LP, G, 1e-3, 10, 0, acc, None)
            torch.cuda.synchronize()
            got = T.cpu().numpy().astype(np.float64)
            acc = acc.cpu().numpy()
    for ci in range(2):
        x0 = th[ci].astype(np.float64)
        lr, gr = t.logp_grad(x0)
        r = ohmc.trajectory(t, x0, lr, gr, 1e-3, 10, 0, int(prob.chain_ids[ci]))
        assert bool(acc[ci]) == r["accepted"]
        assert np.linalg.norm(got[ci] - r["theta"]) <= 1e-4 * np.linalg.norm(r["theta"])


def test_masked_wgrad_sensitivity_mode():
    """Squared-operand mode (hmc_sensitivity) through the masked kernel: the oracle's S_i^2."""
    from paper_2507_14652_b200 import abi
    arch, kw, seed = CASES["deeponet"]
    prob = make_tiny_problem(arch, n_chains=1, seed=seed, noise=0.3, **kw)
    with _Mode(4):
        got = abi.hmc_sensitivity(prob)
    ref = osens.sensitivities(prob.arch, prob.frozen.astype(np.float64), prob.sigma_vi.astype(np.float64),
                              {"u": prob.u, "q": prob.q, "v": prob.v})
    assert np.linalg.norm(got - ref) / np.linalg.norm(ref) <= 1e-5
    big = ref >= 1e-3 * ref.max()
    assert np.max(np.abs(got[big] - ref[big]) / ref[big]) <= 1e-5
