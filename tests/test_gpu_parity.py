"""GPU <-> oracle parity through the C-ABI (SURVEY §8(c) parity protocol).

Every case runs the CUDA path via paper_2507_14652_b200.abi and the fp64 oracle on the same
seeded inputs and Philox streams."""
import math

import numpy as np
import pytest

from hmcdata import ArchSpec, NetSpec, make_problem, make_tiny_problem
from oracle import hmc as ohmc
from oracle import philox as ophilox

from gpu_util import (KAPPA_Q26B, STATE_RTOL, assert_grad_close, assert_grad_elementwise, gpu_grad, jittered_states,
                      to_dev, torch_cuda)

pytestmark = pytest.mark.gpu


def _ctx(prob, **kw):
    from paper_2507_14652_b200 import abi
    return abi.Context(prob, **kw)


# ------------------------------------------------------------------------------------ RNG ---
def test_philox_words_bitwise_1M():
    from paper_2507_14652_b200 import abi
    torch = torch_cuda()
    nb = 1 << 18   # 2^18 blocks = 1,048,576 words
    for (seed, tag, it, ch) in [(0, 0, 0, 0), (3, 0, 17, 5), ((7 << 32) + 11, 1, 4096, 63)]:
        out = torch.empty(nb * 4, dtype=torch.int32, device="cuda")
        abi.hmc_philox_words(seed, tag, it, ch, nb, out)
        got = out.cpu().numpy().view(np.uint32).reshape(nb, 4)
        np.testing.assert_array_equal(got, ophilox.words(seed, tag, it, ch, nb))


def test_momentum_matches_oracle():
    prob = make_tiny_problem(ArchSpec("mlp", (NetSpec.plain((2, 9, 1)),)), n=10, n_chains=3,
                             seed=1, inv_mass=True)
    prob.chain_ids = np.array([4, 9, 1], dtype=np.uint32)
    with _ctx(prob) as c:
        p = np.empty((3, prob.k), dtype=np.float32)
        from paper_2507_14652_b200 import abi
        abi.hmc_momentum(c.ctx, 77, p)
    t = ohmc.Target(prob)
    for ci, ch in enumerate(prob.chain_ids):
        ref = ohmc.momentum(t, 77, int(ch))
        np.testing.assert_allclose(p[ci], ref, rtol=2e-7, atol=1e-7)


# ----------------------------------------------------------------------------- gradients ---
TINY = {
    "mlp_ragged": (ArchSpec("mlp", (NetSpec.plain((3, 150, 70, 1)),)), dict(n=333, active_frac=0.6)),
    "mlp_sin_nobias": (ArchSpec("mlp", (NetSpec((2, 40, 33, 1), ("sin", "tanh", "identity"),
                                                 (True, False, True)),)), dict(n=97, active_frac=0.8)),
    "mlp_deep_narrow": (ArchSpec("mlp", (NetSpec.plain((1, 20, 20, 20, 1)),)), dict(n=64, active_frac=1.0)),
    "deeponet_ragged": (ArchSpec("deeponet", (NetSpec.plain((7, 130, 64, 50)),
                                              NetSpec.plain((3, 70, 50), last="tanh")), has_b0=True),
                        dict(n_c=150, n_x=201, active_frac=0.5)),
    # few query points, many conditions: the dT = R^T B GEMM splits K into 2 row slabs (dt_ksplit)
    "deeponet_dt_ksplit": (ArchSpec("deeponet", (NetSpec.plain((7, 64, 40)),
                                                 NetSpec.plain((3, 70, 40), last="tanh")), has_b0=True),
                           dict(n_c=300, n_x=70, active_frac=0.5)),
    "deeponet_sin": (ArchSpec("deeponet", (NetSpec((4, 20, 12), ("sin", "identity"), (True, True)),
                                           NetSpec((2, 16, 12), ("tanh", "sin"), (True, False))),
                              has_b0=False), dict(n_c=33, n_x=65, active_frac=0.9)),
}


# fixed per-case seeds (reproducible across processes, unlike salted str hashes)
TINY_SEED = {"mlp_ragged": 21, "mlp_sin_nobias": 22, "mlp_deep_narrow": 23, "deeponet_ragged": 24,
             "deeponet_sin": 25, "deeponet_dt_ksplit": 26}


@pytest.mark.parametrize("name", sorted(TINY))
def test_grad_tiny(name):
    arch, kw = TINY[name]
    prob = make_tiny_problem(arch, n_chains=3, seed=TINY_SEED[name], noise=0.3, **kw)
    th = jittered_states(prob, 3)
    with _ctx(prob) as c:
        if name == "deeponet_dt_ksplit":
            from paper_2507_14652_b200 import abi
            assert "dT K split 2" in abi.hmc_engine_info(c.ctx), abi.hmc_engine_info(c.ctx)
        lp, g = gpu_grad(c, th)
    t = ohmc.Target(prob)
    for ci in range(3):
        lr, gr = t.logp_grad(th[ci])
        assert_grad_close(lp[ci], g[ci], lr, gr, f"{name} chain {ci}")


@pytest.fixture
def simt_engine():
    """Contexts set up inside the test run every GEMM on the SIMT engine (hmc_debug_set_engine)."""
    from paper_2507_14652_b200 import abi
    abi.hmc_debug_set_engine(1)
    yield
    abi.hmc_debug_set_engine(0)


@pytest.mark.parametrize("name", ["mlp_ragged", "deeponet_ragged"])
def test_grad_simt_engine_forced(name, simt_engine):
    """The SIMT engine alone meets the same tolerances."""
    arch, kw = TINY[name]
    prob = make_tiny_problem(arch, n_chains=2, seed=11, noise=0.3, **kw)
    th = jittered_states(prob, 2)
    with _ctx(prob) as c:
        from paper_2507_14652_b200 import abi
        assert abi.hmc_engine_info(c.ctx).split(" + ")[0] == "simt"
        lp, g = gpu_grad(c, th)
    t = ohmc.Target(prob)
    for ci in range(2):
        lr, gr = t.logp_grad(th[ci])
        assert_grad_close(lp[ci], g[ci], lr, gr, name)


def test_grad_cfg5_engines_agree():
    """cfg5 gradient: tcgen05 engine vs SIMT engine vs oracle (chain 0)."""
    from paper_2507_14652_b200 import abi
    prob = make_problem("cfg5", n_chains=4)
    th = jittered_states(prob, 4)
    with _ctx(prob) as c:
        assert "tcgen05" in abi.hmc_engine_info(c.ctx)
        lp_tc, g_tc = gpu_grad(c, th)
    abi.hmc_debug_set_engine(1)
    try:
        with _ctx(prob) as c:
            assert abi.hmc_engine_info(c.ctx).split(" + ")[0] == "simt"
            lp_s, g_s = gpu_grad(c, th)
    finally:
        abi.hmc_debug_set_engine(0)
    t = ohmc.Target(prob)
    lr, gr = t.logp_grad(th[0])
    assert_grad_close(lp_tc[0], g_tc[0], lr, gr, "tc")
    assert_grad_close(lp_s[0], g_s[0], lr, gr, "simt")


def test_grad_case1_sine_and_blr():
    case1 = ArchSpec("mlp", (NetSpec((1, 2, 1), ("sin", "identity"), (True, False)),))
    for prob in (make_tiny_problem(case1, n=20, seed=4, noise=0.1), make_problem("blr", n_chains=2)):
        th = jittered_states(prob, prob.n_chains)
        with _ctx(prob) as c:
            lp, g = gpu_grad(c, th)
        t = ohmc.Target(prob)
        for ci in range(prob.n_chains):
            lr, gr = t.logp_grad(th[ci])
            assert_grad_close(lp[ci], g[ci], lr, gr, prob.name)


def test_grad_mask_upper_layers_only():
    """l_min > 0: no weight gradient below the lowest active layer, input grads stop there."""
    arch = ArchSpec("mlp", (NetSpec.plain((2, 30, 30, 1)),))
    prob = make_tiny_problem(arch, n=50, seed=5)
    # active = a few entries of layer 2 (flat offsets after layer 0: 2*30+30 = 90, layer 1 W 90..989)
    prob.idx = np.array([95, 300, 989, 1000, 1019], dtype=np.int32)
    th = jittered_states(prob, 2)
    with _ctx(prob, n_chains=2) as c:
        lp, g = gpu_grad(c, th)
    t = ohmc.Target(prob)
    for ci in range(2):
        lr, gr = t.logp_grad(th[ci])
        assert_grad_close(lp[ci], g[ci], lr, gr)


def test_grad_deeponet_trunk_only_mask():
    arch = ArchSpec("deeponet", (NetSpec.plain((5, 24, 16)), NetSpec.plain((2, 24, 16), last="tanh")),
                    has_b0=True)
    prob = make_tiny_problem(arch, n_c=40, n_x=70, seed=6)
    Pb = 5 * 24 + 24 + 24 * 16 + 16
    prob.idx = np.arange(Pb, prob.P, 3, dtype=np.int32)    # trunk + maybe b0, no branch entry
    th = jittered_states(prob, 2)
    with _ctx(prob, n_chains=2) as c:
        lp, g = gpu_grad(c, th)
    t = ohmc.Target(prob)
    for ci in range(2):
        lr, gr = t.logp_grad(th[ci])
        assert_grad_close(lp[ci], g[ci], lr, gr)


@pytest.mark.parametrize("cfg,check", [("cfg1", 1), ("cfg2", 3), ("cfg3", 2), ("cfg4", 2), ("cfg5", 2)])
def test_grad_full_configs(cfg, check):
    """Full BASELINE sizes in the bench launch configuration (all C chains batched); the oracle
    checks `check` sampled chains (seeded init for chain 0, jittered states otherwise)."""
    prob = make_problem(cfg)
    th = jittered_states(prob, prob.n_chains)
    with _ctx(prob) as c:
        lp, g = gpu_grad(c, th)
    t = ohmc.Target(prob)
    chains = sorted(set([0] + list(np.linspace(1, prob.n_chains - 1, max(check - 1, 1)).astype(int))))[:check]
    for ci in chains:
        lr, gr = t.logp_grad(th[ci])
        assert_grad_close(lp[ci], g[ci], lr, gr, f"{cfg} chain {ci}")


# --------------------------------------------------------------------------- trajectories ---
def _gpu_traj(c, th, lp, g, eps, L, it):
    torch = torch_cuda()
    from paper_2507_14652_b200 import abi
    C = th.shape[0]
    T = to_dev(th, torch.float32)
    LP = to_dev(lp, torch.float64)
    G = to_dev(g, torch.float32)
    acc = torch.zeros(C, dtype=torch.uint8, device="cuda")
    dH = torch.zeros(C, dtype=torch.float64, device="cuda")
    abi.hmc_trajectory(c.ctx, T, LP, G, eps, L, it, acc, dH)
    torch.cuda.synchronize()
    return T.cpu().numpy(), LP.cpu().numpy(), G.cpu().numpy(), acc.cpu().numpy(), dH.cpu().numpy()


def _check_traj(prob, th, eps, L, it, chains, decision_margin=0.0):
    with _ctx(prob) as c:
        lp, g = gpu_grad(c, th)
        T1, LP1, G1, acc, dH = _gpu_traj(c, th, lp, g, eps, L, it)
    t = ohmc.Target(prob)
    for ci in chains:
        ch = int(prob.chain_ids[ci])
        lr, gr = t.logp_grad(th[ci])
        r = ohmc.trajectory(t, th[ci].astype(np.float64), lr, gr, eps, L, it, ch)
        if not np.isfinite(r["dH"]) or abs(r["dH"]) > 1e6 * max(1.0, abs(r["H0"])):
            # divergent trajectory (leapfrog unstable at this eps): both sides must reject
            assert not r["accepted"] and not acc[ci], (ci, r["dH"], dH[ci])
            np.testing.assert_array_equal(T1[ci], th[ci])
            continue
        tol_dH = 1e-6 * (abs(r["H0"]) + abs(r["H1"])) + 1e-4
        assert abs(dH[ci] - r["dH"]) <= tol_dH, (ci, dH[ci], r["dH"])
        margin = abs(math.log(r["u"]) - (r["H0"] - r["H1"]))
        if margin > max(decision_margin, 2 * tol_dH):
            assert bool(acc[ci]) == r["accepted"], (ci, margin)
        if acc[ci] and r["accepted"]:
            ref = r["theta_prop"]
            disp = np.linalg.norm(ref - th[ci])
            err = np.linalg.norm(T1[ci] - ref)
            assert err <= STATE_RTOL * np.linalg.norm(ref), (ci, err / np.linalg.norm(ref))
            assert err <= 2e-3 * max(disp, 1e-30) + 1e-6, (ci, err, disp)
        elif not acc[ci]:
            np.testing.assert_array_equal(T1[ci], th[ci])
    return acc, dH


def stable_eps(prob, th, frac=0.25, iters=20):
    """frac x the leapfrog stability limit 2/sqrt(lambda_max(M^-1 H)) at th (oracle power
    iteration with finite-difference Hessian-vector products)."""
    t = ohmc.Target(prob)
    x = th.astype(np.float64)
    v = np.random.default_rng(0).normal(size=prob.k)
    v /= np.linalg.norm(v)
    im = t.inv_mass
    lam, h = 1.0, 1e-5
    for _ in range(iters):
        Hv = -im * (t.logp_grad(x + h * v)[1] - t.logp_grad(x - h * v)[1]) / (2 * h)
        lam = abs(v @ Hv)
        v = Hv / np.linalg.norm(Hv)
    return frac * 2.0 / math.sqrt(lam)


def test_trajectory_tiny_configs():
    for name in ("mlp_ragged", "deeponet_ragged", "mlp_sin_nobias"):
        arch, kw = TINY[name]
        prob = make_tiny_problem(arch, n_chains=3, seed=7, noise=0.3, inv_mass=True, **kw)
        th = jittered_states(prob, 3, scale=0.01)
        eps = stable_eps(prob, th[0])
        _check_traj(prob, th, eps, 15, 3, range(3))
        # an unstable step size: divergent proposals must be rejected on both sides
        _check_traj(prob, th, 40 * eps, 15, 4, range(3))


def test_trajectory_cfg1_resynced_all_200():
    """cfg1: all 200 trajectories (L = 20) re-synced to the oracle's start state."""
    prob = make_problem("cfg1")
    t = ohmc.Target(prob)
    th = prob.frozen[prob.idx].astype(np.float64)
    lp, g = t.logp_grad(th)
    states = []
    for s in range(200):
        states.append(th.astype(np.float32))
        r = ohmc.trajectory(t, th, lp, g, prob.eps, prob.L, s, 0)
        th, lp, g = r["theta"], r["logp"], r["grad"]
    from paper_2507_14652_b200 import abi
    n_bad = 0
    with _ctx(prob) as c:
        for s in range(0, 200, 1):
            th32 = states[s][None, :]
            lpg, gg = gpu_grad(c, th32)
            T1, _, _, acc, dH = _gpu_traj(c, th32, lpg, gg, prob.eps, prob.L, s)
            lr, gr = t.logp_grad(th32[0].astype(np.float64))
            r = ohmc.trajectory(t, th32[0].astype(np.float64), lr, gr, prob.eps, prob.L, s, 0)
            n_bad += int(bool(acc[0]) != r["accepted"])
            if acc[0] and r["accepted"]:
                ref = r["theta_prop"]
                assert np.linalg.norm(T1[0] - ref) <= STATE_RTOL * np.linalg.norm(ref)
    assert n_bad == 0


def test_cfg1_gradients_at_every_20th_chain_state():
    """Q26 at states the chain visits: the oracle's free-running cfg1 chain (200 samples), every
    20th state: GPU log pi and gradient vs the oracle, element-wise |dg_i| <= 1e-5 S_i."""
    prob = make_problem("cfg1")
    t = ohmc.Target(prob)
    th0 = prob.frozen[prob.idx].astype(np.float64)
    ref_s, _, _ = ohmc.sample_chain(t, th0, prob.eps, prob.L, 0, prob.S, 0)
    states = np.stack([ref_s[s] for s in range(19, prob.S, 20)]).astype(np.float32)   # 10 states
    with _ctx(prob) as c:
        for i, st in enumerate(states):
            lp, g = gpu_grad(c, st[None, :])
            x = st.astype(np.float64)
            lr, gr = t.logp_grad(x)
            assert_grad_elementwise(lp[0], g[0], lr, gr, t.grad_scale(x, KAPPA_Q26B), f"cfg1 state {20 * i + 19}")


def test_cfg2_resynced_20_trajectories_8_chains():
    """the first 20 trajectories of each of the 8 chains (L = 50), re-synced
    (each starts from the oracle's state rounded to fp32): log pi and gradient element-wise at every
    visited state (Q26), identical decisions outside the rounding margin, end states within 1e-4."""
    prob = make_problem("cfg2")
    t = ohmc.Target(prob)
    C, nt = prob.n_chains, 20
    starts, refs = np.empty((nt, C, prob.k), dtype=np.float32), [[None] * C for _ in range(nt)]
    for ci in range(C):
        th = prob.frozen[prob.idx].astype(np.float64)
        for s in range(nt):
            th32 = th.astype(np.float32)
            x = th32.astype(np.float64)
            lr, gr = t.logp_grad(x)
            r = ohmc.trajectory(t, x, lr, gr, prob.eps, prob.L, s, ci)
            starts[s, ci] = th32
            refs[s][ci] = (lr, gr, r)
            th = r["theta"]
    n_acc = 0
    with _ctx(prob) as c:
        for s in range(nt):
            lp, g = gpu_grad(c, starts[s])
            T1, _, _, acc, dH = _gpu_traj(c, starts[s], lp, g, prob.eps, prob.L, s)
            for ci in range(C):
                lr, gr, r = refs[s][ci]
                x = starts[s, ci].astype(np.float64)
                assert_grad_elementwise(lp[ci], g[ci], lr, gr, t.grad_scale(x, KAPPA_Q26B), f"traj {s} chain {ci}")
                # dH = H* - H0: each log pi within the north_star 1e-5 relative (the kinetic terms
                # follow the end state, within 1e-4 relative, and are far smaller here)
                tol_dH = 1e-5 * (abs(lr) + abs(r["logp"] if r["accepted"] else r["H1"])) + 1e-4
                assert abs(dH[ci] - r["dH"]) <= tol_dH, (s, ci, dH[ci], r["dH"])
                if abs(np.log(r["u"]) - (r["H0"] - r["H1"])) > 2 * tol_dH:
                    assert bool(acc[ci]) == r["accepted"], (s, ci)
                if acc[ci] and r["accepted"]:
                    n_acc += 1
                    ref = r["theta_prop"]
                    assert np.linalg.norm(T1[ci] - ref) <= STATE_RTOL * np.linalg.norm(ref), (s, ci)
    assert n_acc >= C * nt // 2


def test_cfg1_free_running_decisions_identical():
    """cfg1 free-running 200 samples (hmc_sample, one graph per trajectory): identical
    accept/reject sequence to the oracle's chain."""
    torch = torch_cuda()
    from paper_2507_14652_b200 import abi
    prob = make_problem("cfg1")
    t = ohmc.Target(prob)
    th0 = prob.frozen[prob.idx].astype(np.float64)
    ref_s, ref_acc, ref_dH = ohmc.sample_chain(t, th0, prob.eps, prob.L, 0, prob.S, 0)
    with _ctx(prob) as c:
        th = th0.astype(np.float32)[None, :]
        lp, g = gpu_grad(c, th)
        T, LP, G = to_dev(th, torch.float32), to_dev(lp, torch.float64), to_dev(g, torch.float32)
        S = prob.S
        samples = torch.empty(1, S, prob.k, dtype=torch.float32, device="cuda")
        acc = torch.empty(1, S, dtype=torch.uint8, device="cuda")
        dH = torch.empty(1, S, dtype=torch.float64, device="cuda")
        abi.hmc_sample(c.ctx, T, LP, G, prob.eps, prob.L, 0, S, samples, acc, dH)
        torch.cuda.synchronize()
    acc = acc.cpu().numpy()[0].astype(bool)
    np.testing.assert_array_equal(acc, ref_acc)
    np.testing.assert_allclose(dH.cpu().numpy()[0], ref_dH, rtol=0, atol=1e-3)
    s = samples.cpu().numpy()[0]
    rel = np.linalg.norm(s - ref_s, axis=1) / np.linalg.norm(ref_s, axis=1)
    assert rel.max() <= 1e-4, rel.max()


# 0.25 x 2/sqrt(lambda_max) at the seeded state (oracle power iteration, DESIGN.md §3 "step
# sizes"): cfg4 lambda_max ~ 5.0e10, cfg5 ~ 3.8e11.  The BASELINE eps of cfg4 / cfg5 is 11x /
# 15x above the stability limit, so at that eps every trajectory diverges and is rejected.
STABLE_EPS = {"cfg2": None, "cfg3": None, "cfg4": 1.1e-6, "cfg5": 4.0e-7}


@pytest.mark.parametrize("cfg,L,which", [("cfg2", 50, "config"), ("cfg3", 50, "config"),
                                         ("cfg4", 50, "config"), ("cfg4", 50, "stable"),
                                         ("cfg5", 50, "config"), ("cfg5", 50, "stable")])
def test_trajectory_full_configs_truncated(cfg, L, which):
    """cfg2-5 at full size with all chains batched; L truncated to 50 (north_star: L <= 50);
    oracle re-runs chains 0 and C-1, at the configured eps and (cfg4/5) a stable eps."""
    prob = make_problem(cfg)
    th = jittered_states(prob, prob.n_chains, scale=0.005)
    eps = prob.eps if which == "config" else STABLE_EPS[cfg]
    _check_traj(prob, th, eps, L, 0, [0, prob.n_chains - 1])


# ----------------------------------------------------------------------- sampler contract ---
def test_L0_identity_and_resume_bitwise():
    torch = torch_cuda()
    from paper_2507_14652_b200 import abi
    arch, kw = TINY["mlp_ragged"]
    prob = make_tiny_problem(arch, n_chains=4, seed=8, noise=0.3, **kw)
    th = jittered_states(prob, 4)
    with _ctx(prob) as c:
        lp, g = gpu_grad(c, th)
        T1, LP1, G1, acc, dH = _gpu_traj(c, th, lp, g, 1e-3, 0, 5)
        np.testing.assert_array_equal(T1, th)
        assert acc.all() and np.all(dH == 0)

        def run(S, it, T, LP, G):
            smp = torch.empty(4, S, prob.k, dtype=torch.float32, device="cuda")
            a = torch.empty(4, S, dtype=torch.uint8, device="cuda")
            abi.hmc_sample(c.ctx, T, LP, G, 1e-3, 7, it, S, smp, a, None)
            return smp.cpu().numpy(), a.cpu().numpy()
        mk = lambda: (to_dev(th, torch.float32), to_dev(lp, torch.float64), to_dev(g, torch.float32))
        T, LP, G = mk()
        s10, a10 = run(10, 100, T, LP, G)
        T, LP, G = mk()
        s5a, a5a = run(5, 100, T, LP, G)
        s5b, a5b = run(5, 105, T, LP, G)
        np.testing.assert_array_equal(s10, np.concatenate([s5a, s5b], axis=1))
        np.testing.assert_array_equal(a10, np.concatenate([a5a, a5b], axis=1))
        assert 0 < a10.mean() <= 1


def test_chain_results_independent_of_batch():
    """A chain's trajectory is bitwise identical whether it runs alone or batched with others
    (batch invariance -> chain mode across GPUs equals the 1-GPU run)."""
    arch, kw = TINY["deeponet_ragged"]
    prob = make_tiny_problem(arch, n_chains=4, seed=9, noise=0.3, **kw)
    prob.chain_ids = np.array([10, 11, 12, 13], dtype=np.uint32)
    th = jittered_states(prob, 4)
    with _ctx(prob) as c:
        lp, g = gpu_grad(c, th)
        T4, LP4, G4, a4, d4 = _gpu_traj(c, th, lp, g, 1e-3, 6, 2)
    single = make_tiny_problem(arch, n_chains=1, seed=9, noise=0.3, **kw)
    single.chain_ids = np.array([12], dtype=np.uint32)
    with _ctx(single) as c:
        lp1, g1 = gpu_grad(c, th[2:3])
        T1, LP1, G1, a1, d1 = _gpu_traj(c, th[2:3], lp1, g1, 1e-3, 6, 2)
    np.testing.assert_array_equal(lp1, lp[2:3])
    np.testing.assert_array_equal(T1[0], T4[2])
    assert a1[0] == a4[2] and d1[0] == d4[2]


def test_blr_gpu_samples_match_closed_form():
    """GPU sampler statistics on the BLR pin config: mean within 4 MCSE, covariance within 10%."""
    torch = torch_cuda()
    from paper_2507_14652_b200 import abi
    from test_oracle_hmc import blr_closed_form, blr_eps
    prob = make_problem("blr", n_chains=4)
    A, mu = blr_closed_form(prob)
    Sigma = np.linalg.inv(A)
    eps = blr_eps(prob, A)
    S = 10000
    with _ctx(prob) as c:
        th = np.zeros((4, 4), dtype=np.float32)
        lp, g = gpu_grad(c, th)
        T, LP, G = to_dev(th, torch.float32), to_dev(lp, torch.float64), to_dev(g, torch.float32)
        smp = torch.empty(4, S, 4, dtype=torch.float32, device="cuda")
        a = torch.empty(4, S, dtype=torch.uint8, device="cuda")
        abi.hmc_sample(c.ctx, T, LP, G, eps, 4, 0, S, smp, a, None)
        torch.cuda.synchronize()
    D = smp.cpu().numpy()[:, 500:, :].reshape(-1, 4).astype(np.float64)
    assert a.float().mean().item() > 0.8
    nb = 40
    bm = np.array_split(D, nb)
    mcse = np.std([b.mean(axis=0) for b in bm], axis=0, ddof=1) / math.sqrt(nb)
    assert np.all(np.abs(D.mean(axis=0) - mu) < 4 * mcse)
    sd = np.sqrt(np.diag(Sigma))
    assert np.max(np.abs(np.cov(D.T) - Sigma) / np.outer(sd, sd)) < 0.10


def test_config_errors_are_reported():
    from paper_2507_14652_b200 import abi
    prob = make_tiny_problem(ArchSpec("mlp", (NetSpec.plain((2, 5, 1)),)), n=8, seed=1)
    bad = [("idx", np.array([3, 2], dtype=np.int32)), ("idx", np.array([0, 10_000], dtype=np.int32)),
           ("noise_sigma", 0.0), ("prior_sigma", -1.0)]
    for field, val in bad:
        p2 = make_tiny_problem(ArchSpec("mlp", (NetSpec.plain((2, 5, 1)),)), n=8, seed=1)
        setattr(p2, field, val)
        with pytest.raises(abi.HmcError) as e:
            abi.Context(p2)
        assert e.value.code == abi.HMC_E_CONFIG
    # world / shard validation: world in {1, 2, 4, 8}, SINGLE needs world 1,
    # DATA mode needs equal shards (more in test_gpu_contract.py)
    for kw in (dict(mode="chain", world=3), dict(mode="single", world=2), dict(mode="data", world=1, n_global=9)):
        with pytest.raises(abi.HmcError) as e:
            abi.Context(prob, **kw)
        assert e.value.code == abi.HMC_E_CONFIG, kw
    with abi.Context(prob) as c:
        th = jittered_states(prob, 1)
        lp, g = gpu_grad(c, th)
        for bad in (dict(eps=-1.0, L=5, it=0), dict(eps=float("nan"), L=5, it=0), dict(eps=1e-3, L=-1, it=0),
                    dict(eps=1e-3, L=5, it=1 << 32), dict(eps=0.0, L=5, it=0)):   # eps 0 before hmc_adapt
            with pytest.raises(abi.HmcError) as e:
                abi.hmc_trajectory(c.ctx, th, lp, g, bad["eps"], bad["L"], bad["it"])
            assert e.value.code == abi.HMC_E_CONFIG, bad


@pytest.mark.parametrize("name", ["mlp_ragged", "deeponet_ragged"])
def test_host_buffers_equal_device_buffers(name):
    """The end-to-end path (hmc_sample on pinned / pageable host buffers, the bench's e2e) gives
    bitwise the same samples, decisions, energies and final state as device buffers."""
    torch = torch_cuda()
    from paper_2507_14652_b200 import abi
    arch, kw = TINY[name]
    prob = make_tiny_problem(arch, n_chains=3, seed=9, noise=0.3, **kw)
    th = jittered_states(prob, 3, scale=0.005)
    S, L, eps = 4, 6, 5e-4
    with _ctx(prob) as c:
        lp, g = gpu_grad(c, th)
        T, LP, G = to_dev(th, torch.float32), to_dev(lp, torch.float64), to_dev(g, torch.float32)
        smp = torch.empty(3, S, prob.k, device="cuda")
        a = torch.empty(3, S, dtype=torch.uint8, device="cuda")
        d = torch.empty(3, S, dtype=torch.float64, device="cuda")
        abi.hmc_sample(c.ctx, T, LP, G, eps, L, 11, S, smp, a, d)
        torch.cuda.synchronize()
        hT, hLP, hG = th.copy(), lp.copy(), g.copy()
        hs = np.empty((3, S, prob.k), dtype=np.float32)
        ha = np.empty((3, S), dtype=np.uint8)
        hd = np.empty((3, S), dtype=np.float64)
        abi.hmc_sample(c.ctx, hT, hLP, hG, eps, L, 11, S, hs, ha, hd)
    np.testing.assert_array_equal(hs, smp.cpu().numpy())
    np.testing.assert_array_equal(ha, a.cpu().numpy())
    np.testing.assert_array_equal(hd, d.cpu().numpy())
    np.testing.assert_array_equal(hT, T.cpu().numpy())
    np.testing.assert_array_equal(hG, G.cpu().numpy())


@pytest.mark.parametrize("name", ["mlp_ragged", "mlp_deep_narrow", "mlp_sin_nobias"])
def test_grad_tiny_per_layer_engines(name):
    """MLPs on the per-layer engines (hmc_debug_set_engine(2): no narrow engine), i.e. through the
    one-pass output layer (k_out_fused; ragged 70 / 20-wide inputs, 333 / 64 rows: partial 256-row
    chunks and 32-row blocks) - and, for the sin layer below the output, the four-kernel path."""
    from paper_2507_14652_b200 import abi
    arch, kw = TINY[name]
    prob = make_tiny_problem(arch, n_chains=3, seed=TINY_SEED[name] + 100, noise=0.3, **kw)
    th = jittered_states(prob, 3)
    abi.hmc_debug_set_engine(2)
    try:
        with _ctx(prob) as c:
            assert not abi.hmc_engine_info(c.ctx).startswith("narrow")
            lp, g = gpu_grad(c, th)
    finally:
        abi.hmc_debug_set_engine(0)
    t = ohmc.Target(prob)
    for ci in range(3):
        lr, gr = t.logp_grad(th[ci])
        assert_grad_close(lp[ci], g[ci], lr, gr, f"{name} per-layer chain {ci}")
