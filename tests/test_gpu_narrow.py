"""The narrow-network engine (csrc/narrow.cuh: one cluster kernel per leapfrog step / trajectory,
weights resident in shared memory; north_star subsystem (1)) against the fp64 oracle, through the
C-ABI, plus the sampler contract on it (resume, batch invariance, L = 0, the per-layer engines
agreeing within tolerance)."""
import numpy as np
import pytest

from hmcdata import ArchSpec, NetSpec, make_problem, make_tiny_problem
from oracle import hmc as ohmc

from gpu_util import STATE_RTOL, assert_grad_close, gpu_grad, jittered_states, to_dev, torch_cuda

pytestmark = pytest.mark.gpu

NARROW = {
    # rows not a multiple of the CTA rows, widths not multiples of 16, 3 inputs
    "ragged": (ArchSpec("mlp", (NetSpec.plain((3, 36, 20, 1)),)), dict(n=333, active_frac=0.6), 41),
    # 128-wide layers (two passes of the 64 x 64 thread grid), few rows per CTA
    "wide128": (ArchSpec("mlp", (NetSpec.plain((2, 128, 128, 1)),)), dict(n=700, active_frac=0.2), 42),
    # identity hidden activation, no bias in the middle layer, 8 inputs (cfg3's input width)
    "ident_nobias": (ArchSpec("mlp", (NetSpec((8, 24, 16, 1), ("identity", "tanh", "identity"),
                                              (True, False, True)),)), dict(n=150, active_frac=0.9), 43),
    # deep: 7 linear layers
    "deep": (ArchSpec("mlp", (NetSpec.plain((1, 16, 16, 16, 16, 16, 16, 1)),)), dict(n=96, active_frac=1.0), 44),
    # tiny data: one CTA per chain (n < 32)
    "tiny_rows": (ArchSpec("mlp", (NetSpec.plain((1, 8, 1)),)), dict(n=5, active_frac=1.0), 45),
}


def _engine(c):
    from paper_2507_14652_b200 import abi
    return abi.hmc_engine_info(c.ctx)


@pytest.mark.parametrize("name", sorted(NARROW))
def test_narrow_grad_matches_oracle(name):
    torch_cuda()
    from paper_2507_14652_b200 import abi
    arch, kw, seed = NARROW[name]
    prob = make_tiny_problem(arch, n_chains=3, seed=seed, noise=0.3, **kw)
    th = jittered_states(prob, 3)
    with abi.Context(prob) as c:
        assert _engine(c).startswith("narrow"), _engine(c)
        lp, g = gpu_grad(c, th)
    t = ohmc.Target(prob)
    for ci in range(3):
        lr, gr = t.logp_grad(th[ci])
        assert_grad_close(lp[ci], g[ci], lr, gr, f"{name} chain {ci}")


def test_narrow_mask_upper_layers_only():
    """l_min > 0: the backward stops at the lowest active layer."""
    torch_cuda()
    from paper_2507_14652_b200 import abi
    prob = make_tiny_problem(ArchSpec("mlp", (NetSpec.plain((2, 32, 32, 1)),)), n=120, seed=46)
    # layer 0: W 0..63, b 64..95; layer 1: W 96..1119, b 1120..1151; output: w 1152..1183, b 1184
    prob.idx = np.array([100, 500, 1119, 1130, 1160, 1184], dtype=np.int32)
    th = jittered_states(prob, 2)
    with abi.Context(prob, n_chains=2) as c:
        assert _engine(c).startswith("narrow")
        lp, g = gpu_grad(c, th)
    t = ohmc.Target(prob)
    for ci in range(2):
        lr, gr = t.logp_grad(th[ci])
        assert_grad_close(lp[ci], g[ci], lr, gr)
    # output layer only (no hidden-layer backward at all)
    prob.idx = np.array([1152, 1170, 1184], dtype=np.int32)
    th = jittered_states(prob, 2)
    with abi.Context(prob, n_chains=2) as c:
        lp, g = gpu_grad(c, th)
    t = ohmc.Target(prob)
    for ci in range(2):
        lr, gr = t.logp_grad(th[ci])
        assert_grad_close(lp[ci], g[ci], lr, gr)


@pytest.mark.parametrize("cfg", ["cfg1", "cfg2"])
def test_narrow_engine_runs_the_narrow_configs(cfg):
    torch_cuda()
    from paper_2507_14652_b200 import abi
    prob = make_problem(cfg)
    with abi.Context(prob) as c:
        assert _engine(c).startswith("narrow"), _engine(c)
        per_grad, base, per_step = abi.hmc_launch_counts(c.ctx)
    assert (per_grad, base, per_step) == (2, 4, 0)   # one kernel for all L steps of a trajectory


def _traj(c, th, lp, g, eps, L, it):
    torch = torch_cuda()
    from paper_2507_14652_b200 import abi
    C = th.shape[0]
    T, LP, G = to_dev(th, torch.float32), to_dev(lp, torch.float64), to_dev(g, torch.float32)
    acc = torch.zeros(C, dtype=torch.uint8, device="cuda")
    dH = torch.zeros(C, dtype=torch.float64, device="cuda")
    abi.hmc_trajectory(c.ctx, T, LP, G, eps, L, it, acc, dH)
    torch.cuda.synchronize()
    return T.cpu().numpy(), LP.cpu().numpy(), G.cpu().numpy(), acc.cpu().numpy(), dH.cpu().numpy()


@pytest.mark.parametrize("name", ["ragged", "wide128", "deep"])
def test_narrow_trajectory_matches_oracle(name):
    """End state, log pi, gradient, dH and decision of one L = 25 trajectory per chain (the fused
    multi-step kernel: weights updated in shared memory between steps) vs the oracle."""
    torch_cuda()
    from paper_2507_14652_b200 import abi
    from test_gpu_parity import stable_eps
    arch, kw, seed = NARROW[name]
    prob = make_tiny_problem(arch, n_chains=3, seed=seed, noise=0.3, inv_mass=True, **kw)
    th = jittered_states(prob, 3, scale=0.01)
    eps = stable_eps(prob, th[0])
    with abi.Context(prob) as c:
        lp, g = gpu_grad(c, th)
        T1, LP1, G1, acc, dH = _traj(c, th, lp, g, eps, 25, 7)
    t = ohmc.Target(prob)
    for ci in range(3):
        lr, gr = t.logp_grad(th[ci].astype(np.float64))
        r = ohmc.trajectory(t, th[ci].astype(np.float64), lr, gr, eps, 25, 7, int(prob.chain_ids[ci]))
        assert abs(dH[ci] - r["dH"]) <= 1e-6 * (abs(r["H0"]) + abs(r["H1"])) + 1e-4, (ci, dH[ci], r["dH"])
        assert bool(acc[ci]) == r["accepted"]
        if r["accepted"]:
            ref = r["theta_prop"]
            assert np.linalg.norm(T1[ci] - ref) <= STATE_RTOL * np.linalg.norm(ref)
            lpe, ge = t.logp_grad(T1[ci].astype(np.float64))
            assert_grad_close(LP1[ci], G1[ci], lpe, ge, f"{name} end state chain {ci}")


def test_narrow_per_step_equals_fused_and_per_layer_agrees():
    """The profiled trajectory (one launch per step, weights reloaded from HBM) is bitwise equal to
    the fused one (weights updated in shared memory); the per-layer engines (hmc_debug_set_engine
    2) agree within the parity tolerance."""
    torch = torch_cuda()
    from paper_2507_14652_b200 import abi
    prob = make_problem("cfg2")
    th = jittered_states(prob, prob.n_chains, scale=0.005)
    runs = []
    for prof in (False, True):
        with abi.Context(prob) as c:
            lp, g = gpu_grad(c, th)
            abi.hmc_profile(c.ctx, prof)
            runs.append(_traj(c, th, lp, g, prob.eps, prob.L, 3))
    for a, b in zip(runs[0], runs[1]):
        np.testing.assert_array_equal(a, b)
    abi.hmc_debug_set_engine(2)
    try:
        with abi.Context(prob) as c:
            assert not _engine(c).startswith("narrow")
            lp2, g2 = gpu_grad(c, th)
    finally:
        abi.hmc_debug_set_engine(0)
    with abi.Context(prob) as c:
        lp1, g1 = gpu_grad(c, th)
    for ci in range(prob.n_chains):
        assert_grad_close(lp1[ci], g1[ci], lp2[ci].astype(np.float64), g2[ci].astype(np.float64), f"chain {ci}")


def test_narrow_resume_batch_invariance_and_L0():
    torch = torch_cuda()
    from paper_2507_14652_b200 import abi
    arch, kw, seed = NARROW["ragged"]
    prob = make_tiny_problem(arch, n_chains=4, seed=seed, noise=0.3, **kw)
    prob.chain_ids = np.array([20, 21, 22, 23], dtype=np.uint32)
    th = jittered_states(prob, 4, scale=0.005)
    eps = 2e-3
    with abi.Context(prob) as c:
        lp, g = gpu_grad(c, th)
        T0, _, _, a0, d0 = _traj(c, th, lp, g, eps, 0, 1)
        np.testing.assert_array_equal(T0, th)
        assert a0.all() and np.all(d0 == 0)

        def run(S, it, T, LP, G):
            smp = torch.empty(4, S, prob.k, dtype=torch.float32, device="cuda")
            a = torch.empty(4, S, dtype=torch.uint8, device="cuda")
            abi.hmc_sample(c.ctx, T, LP, G, eps, 9, it, S, smp, a, None)
            return smp.cpu().numpy(), a.cpu().numpy()
        mk = lambda: (to_dev(th, torch.float32), to_dev(lp, torch.float64), to_dev(g, torch.float32))
        s8, a8 = run(8, 50, *mk())
        T, LP, G = mk()
        s4a, a4a = run(4, 50, T, LP, G)
        s4b, a4b = run(4, 54, T, LP, G)
        np.testing.assert_array_equal(s8, np.concatenate([s4a, s4b], axis=1))
        np.testing.assert_array_equal(a8, np.concatenate([a4a, a4b], axis=1))
        T4, LP4, G4, acc4, dH4 = _traj(c, th, lp, g, eps, 9, 2)
    single = make_tiny_problem(arch, n_chains=1, seed=seed, noise=0.3, **kw)
    single.chain_ids = np.array([22], dtype=np.uint32)
    with abi.Context(single) as c:
        lp1, g1 = gpu_grad(c, th[2:3])
        T1, LP1, G1, acc1, dH1 = _traj(c, th[2:3], lp1, g1, eps, 9, 2)
    np.testing.assert_array_equal(lp1, lp[2:3])
    np.testing.assert_array_equal(g1, g[2:3])
    np.testing.assert_array_equal(T1[0], T4[2])
    assert acc1[0] == acc4[2] and dH1[0] == dH4[2]


def test_narrow_grid_and_cluster_modes_bitwise_equal():
    """cfg2's 8 chains do not fit as co-resident 16-CTA clusters (7 per GPU), so the batch runs the
    grid mode (cooperative launch, exchanges through L2); a single chain runs the planner's own
    choice and - forced with hmc_debug_set_engine(3) - one cluster (distributed shared memory).  Every sum over data rows is fixed by the row blocks, so chain 3's gradient,
    trajectory and decision are bitwise the same in all three."""
    torch = torch_cuda()
    from paper_2507_14652_b200 import abi
    prob = make_problem("cfg2")
    th = jittered_states(prob, prob.n_chains, scale=0.005)
    with abi.Context(prob) as c:
        assert "grid" in _engine(c), _engine(c)
        lp, g = gpu_grad(c, th)
        T8, LP8, G8, a8, d8 = _traj(c, th, lp, g, prob.eps, prob.L, 5)
    one = make_problem("cfg2", n_chains=1)
    one.chain_ids = np.array([3], dtype=np.uint32)
    for forced in (0, 3):
        abi.hmc_debug_set_engine(forced)
        try:
            with abi.Context(one) as c:
                if forced:
                    assert "cluster" in _engine(c), _engine(c)
                lp1, g1 = gpu_grad(c, th[3:4])
                T1, LP1, G1, a1, d1 = _traj(c, th[3:4], lp1, g1, prob.eps, prob.L, 5)
        finally:
            abi.hmc_debug_set_engine(0)
        np.testing.assert_array_equal(lp1, lp[3:4])
        np.testing.assert_array_equal(g1, g[3:4])
        np.testing.assert_array_equal(T1[0], T8[3])
        np.testing.assert_array_equal(G1[0], G8[3])
        assert a1[0] == a8[3] and d1[0] == d8[3]
