"""DATA mode on one GPU (world = 1): the row layout and the POINTS_XB layout (SURVEY §8(b):
all-gather of the branch outputs, reduce-scatter of dB, both as in-graph NCCL collectives over a
communicator of one) against the oracle and against SINGLE mode.  The world-2 exchange algebra
is covered under gloo in tests/test_dist_cpu.py."""
import numpy as np
import pytest

from hmcdata import ArchSpec, NetSpec, make_problem, make_tiny_problem
from oracle import hmc as ohmc

from gpu_util import assert_grad_close, gpu_grad, jittered_states, torch_cuda

pytestmark = pytest.mark.gpu

ARCH = ArchSpec("deeponet", (NetSpec.plain((7, 130, 64, 50)), NetSpec.plain((3, 70, 50), last="tanh")), has_b0=True)


@pytest.mark.parametrize("shard", ["rows", "points_xb", "points_xc"])
def test_data_mode_world1_grad(shard):
    torch_cuda()
    from paper_2507_14652_b200 import dist as pdist
    prob = make_tiny_problem(ARCH, n_c=40, n_x=37, active_frac=0.5, n_chains=3, seed=51, noise=0.3)
    th = jittered_states(prob, 3)
    from paper_2507_14652_b200 import abi
    with abi.Context(prob, mode="data", shard=shard) as c:   # world = 1
        lp, g = gpu_grad(c, th)
    with abi.Context(prob) as c1:
        lp1, g1 = gpu_grad(c1, th)
    t = ohmc.Target(prob)
    for ci in range(3):
        lr, gr = t.logp_grad(th[ci])
        assert_grad_close(lp[ci], g[ci], lr, gr, f"{shard} chain {ci}")
    np.testing.assert_allclose(lp, lp1, rtol=1e-6)
    assert np.linalg.norm(g - g1) <= 1e-6 * np.linalg.norm(g1)


def test_points_xb_world1_cfg5_and_trajectory():
    """cfg5 at full size (2 chains) in the POINTS_XB layout, and a short trajectory."""
    torch_cuda()
    from paper_2507_14652_b200 import dist as pdist
    from test_gpu_parity import _gpu_traj
    prob = make_problem("cfg5", n_chains=2)
    th = jittered_states(prob, 2)
    t = ohmc.Target(prob)
    with pdist.make_context(prob, "data", 0, 1, shard="points_xb") as c:
        lp, g = gpu_grad(c, th)
        T1, _, _, acc, dH = _gpu_traj(c, th, lp, g, 4.0e-7, 3, 0)
    lr, gr = t.logp_grad(th[0])
    assert_grad_close(lp[0], g[0], lr, gr, "cfg5 points_xb")
    r = ohmc.trajectory(t, th[0].astype(np.float64), lr, gr, 4.0e-7, 3, 0, 0)
    assert abs(dH[0] - r["dH"]) <= 1e-6 * (abs(r["H0"]) + abs(r["H1"])) + 1e-4


def test_points_xb_config_errors():
    torch_cuda()
    from paper_2507_14652_b200 import abi
    prob = make_tiny_problem(ARCH, n_c=8, n_x=6, n_chains=1, seed=52, unaligned=True)
    with pytest.raises(abi.HmcError):
        abi.Context(prob, mode="data", shard="points_xb")


def test_points_xc_world1_cfg5_trajectory():
    """cfg5 at full size (4 chains) in the POINTS_XC layout with real in-graph NCCL collectives
    (a communicator of one), gradient and a short trajectory against the oracle."""
    torch_cuda()
    from paper_2507_14652_b200 import dist as pdist
    from test_gpu_parity import _gpu_traj
    prob = make_problem("cfg5", n_chains=4)
    th = jittered_states(prob, 4)
    t = ohmc.Target(prob)
    with pdist.make_context(prob, "data", 0, 1, shard="points_xc") as c:
        lp, g = gpu_grad(c, th)
        T1, _, _, acc, dH = _gpu_traj(c, th, lp, g, 4.0e-7, 3, 0)
    lr, gr = t.logp_grad(th[0])
    assert_grad_close(lp[0], g[0], lr, gr, "cfg5 points_xc")
    r = ohmc.trajectory(t, th[0].astype(np.float64), lr, gr, 4.0e-7, 3, 0, 0)
    assert abs(dH[0] - r["dH"]) <= 1e-6 * (abs(r["H0"]) + abs(r["H1"])) + 1e-4
