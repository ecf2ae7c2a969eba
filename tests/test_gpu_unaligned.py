"""Unaligned DeepONet on the GPU (per-pair trunk inputs) against the fp64
oracle: gradients (north_star tolerances), a trajectory, the posterior predictive, and the cfg4u
workload at full size.  The trunk runs on n_c * n_x inputs through the same layer engines; the
combine is the row-wise kernel k_pair_combine, the output gradients k_pair_dB / k_pair_dT."""
import numpy as np
import pytest

from hmcdata import ArchSpec, NetSpec, make_problem, make_tiny_problem
from oracle import hmc as ohmc

from gpu_util import assert_grad_close, gpu_grad, jittered_states, torch_cuda

pytestmark = pytest.mark.gpu

ARCHS = {
    # wide enough for the tensor-core engine, ragged widths / counts
    "tc_ragged": (ArchSpec("deeponet", (NetSpec.plain((7, 130, 64, 50)), NetSpec.plain((3, 70, 50), last="tanh")),
                           has_b0=True), dict(n_c=37, n_x=23, active_frac=0.5)),
    # sin layers, no b0, narrow (SIMT engine)
    "sin_narrow": (ArchSpec("deeponet", (NetSpec((4, 20, 12), ("sin", "identity"), (True, True)),
                                         NetSpec((2, 16, 12), ("tanh", "sin"), (True, False))), has_b0=False),
                   dict(n_c=11, n_x=9, active_frac=0.9)),
}


def _ctx(prob):
    from paper_2507_14652_b200 import abi
    return abi.Context(prob)


@pytest.mark.parametrize("name", sorted(ARCHS))
def test_unaligned_grad_tiny(name):
    arch, kw = ARCHS[name]
    prob = make_tiny_problem(arch, n_chains=3, seed=21, noise=0.3, unaligned=True, **kw)
    assert prob.q.ndim == 3
    th = jittered_states(prob, 3)
    with _ctx(prob) as c:
        lp, g = gpu_grad(c, th)
    t = ohmc.Target(prob)
    for ci in range(3):
        lr, gr = t.logp_grad(th[ci])
        assert_grad_close(lp[ci], g[ci], lr, gr, f"{name} chain {ci}")


def test_unaligned_shared_points_equal_aligned_gpu():
    """Every function given the same points: the unaligned path reproduces the aligned one."""
    arch, kw = ARCHS["tc_ragged"]
    al = make_tiny_problem(arch, n_chains=2, seed=22, noise=0.3, **kw)
    un = make_tiny_problem(arch, n_chains=2, seed=22, noise=0.3, **kw)
    un.q = np.ascontiguousarray(np.repeat(al.q[None], al.u.shape[0], 0))
    th = jittered_states(al, 2)
    with _ctx(al) as c:
        la, ga = gpu_grad(c, th)
    with _ctx(un) as c:
        lu, gu = gpu_grad(c, th)
    np.testing.assert_allclose(lu, la, rtol=2e-6)
    assert np.linalg.norm(gu - ga) <= 2e-6 * np.linalg.norm(ga)


def test_unaligned_trajectory_tiny():
    from test_gpu_parity import _check_traj, stable_eps
    arch, kw = ARCHS["tc_ragged"]
    prob = make_tiny_problem(arch, n_chains=3, seed=23, noise=0.3, inv_mass=True, unaligned=True, **kw)
    th = jittered_states(prob, 3, scale=0.01)
    eps = stable_eps(prob, th[0])
    _check_traj(prob, th, eps, 15, 2, range(3))


def test_unaligned_predict():
    torch_cuda()
    from paper_2507_14652_b200 import abi
    arch, kw = ARCHS["tc_ragged"]
    prob = make_tiny_problem(arch, n_chains=4, seed=24, unaligned=True, **kw)
    g = np.random.default_rng(6)
    base = prob.frozen[prob.idx].astype(np.float64)
    samples = (base[None, :] + 0.05 * g.normal(size=(9, prob.k))).astype(np.float32)
    with abi.Context(prob) as c:
        m, v = abi.hmc_predict(c, samples)
    mr, vr = ohmc.predictive(ohmc.Target(prob), samples.astype(np.float64))
    scale = np.abs(mr).max()
    np.testing.assert_allclose(m, mr, rtol=1e-5, atol=1e-6 * scale)
    np.testing.assert_allclose(v, vr, rtol=1e-3, atol=1e-6 * scale * scale)


def test_unaligned_sensitivity_rejected():
    torch_cuda()
    from paper_2507_14652_b200 import abi
    arch, kw = ARCHS["sin_narrow"]
    prob = make_tiny_problem(arch, n_chains=1, seed=25, unaligned=True, **kw)
    with pytest.raises(abi.HmcError):
        abi.hmc_sensitivity(prob)


def test_cfg4u_full_size_grad():
    """cfg4u (1000 functions x 100 per-function points: trunk on 100,000 inputs per chain),
    16 chains batched; chains 0 and 15 against the oracle."""
    prob = make_problem("cfg4u")
    th = jittered_states(prob, prob.n_chains)
    with _ctx(prob) as c:
        lp, g = gpu_grad(c, th)
    t = ohmc.Target(prob)
    for ci in (0, prob.n_chains - 1):
        lr, gr = t.logp_grad(th[ci])
        assert_grad_close(lp[ci], g[ci], lr, gr, f"cfg4u chain {ci}")
