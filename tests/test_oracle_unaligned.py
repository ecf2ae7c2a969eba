"""Pins for the unaligned DeepONet in the oracle (CPU, -m "not gpu").

Unaligned: q [n_c, n_x, d_t], pair (c, x) is F(u_c, y_{c,x}) = sum_k B_k(u_c) T_k(y_{c,x}) + b0
(S:127).  Each pin ties the new code path to something else: the aligned layout (pinned in
test_oracle_network.py) when every function shares its points, pair-by-pair evaluation of the
definition, central finite differences, and the sensitivity definition."""
import numpy as np

from hmcdata import ArchSpec, NetSpec, make_problem, make_tiny_problem
from oracle import hmc as ohmc
from oracle import network as onet
from oracle import sensitivity as osens

ARCH = ArchSpec("deeponet", (NetSpec.plain((4, 7, 5)), NetSpec.plain((2, 6, 5), last="tanh")), has_b0=True)


def _shared(pr):
    """The unaligned layout of an aligned problem: every function gets the same points."""
    n_c = pr.u.shape[0]
    return {"u": pr.u.astype(np.float64), "q": np.repeat(pr.q[None].astype(np.float64), n_c, 0),
            "v": pr.v.astype(np.float64)}


def test_shared_points_reduce_to_aligned():
    pr = make_tiny_problem(ARCH, n_c=6, n_x=9, seed=3)
    th = pr.frozen.astype(np.float64)
    al = {"u": pr.u.astype(np.float64), "q": pr.q.astype(np.float64), "v": pr.v.astype(np.float64)}
    un = _shared(pr)
    np.testing.assert_allclose(onet.predict(ARCH, th, un), onet.predict(ARCH, th, al), rtol=1e-13, atol=1e-13)
    la, ga, _ = onet.loglik_grad(ARCH, th, al, 0.3)
    lu, gu, _ = onet.loglik_grad(ARCH, th, un, 0.3)
    assert abs(lu - la) <= 1e-12 * abs(la)
    np.testing.assert_allclose(gu, ga, rtol=1e-11, atol=1e-11 * np.abs(ga).max())
    np.testing.assert_allclose(onet.grad_abs_scale(ARCH, th, un, 0.3), onet.grad_abs_scale(ARCH, th, al, 0.3),
                               rtol=1e-11)


def test_unaligned_equals_pairwise_definition():
    pr = make_tiny_problem(ARCH, n_c=5, n_x=7, seed=8, unaligned=True)
    assert pr.q.shape == (5, 7, 2)
    th = pr.frozen.astype(np.float64)
    data = {"u": pr.u.astype(np.float64), "q": pr.q.astype(np.float64)}
    F = onet.predict(ARCH, th, data)
    cc, xx = np.meshgrid(np.arange(5), np.arange(7), indexing="ij")
    Fp = onet.predict_pairwise(ARCH, th, data["u"][cc.ravel()], data["q"][cc.ravel(), xx.ravel()])
    np.testing.assert_allclose(F.ravel(), Fp, rtol=1e-13, atol=1e-13)


def test_unaligned_fd_gradient():
    pr = make_tiny_problem(ARCH, n_c=6, n_x=8, active_frac=0.7, seed=9, noise=0.5, unaligned=True)
    tgt = ohmc.Target(pr)
    g = np.random.default_rng(0)
    th = pr.frozen[pr.idx].astype(np.float64) + 0.05 * g.normal(size=pr.k)
    _, grad = tgt.logp_grad(th)
    h = 1e-6
    for j in g.choice(pr.k, size=20, replace=False):
        e = np.zeros(pr.k)
        e[j] = h
        fd = (tgt.logp_grad(th + e)[0] - tgt.logp_grad(th - e)[0]) / (2 * h)
        scale = max(abs(grad[j]), 1e-3 * np.max(np.abs(grad)))
        assert abs(fd - grad[j]) / scale < 1e-5, (j, fd, grad[j])


def test_unaligned_swapping_points_between_functions():
    """Permuting the query points of one function permutes only that row of F (the trunk
    input of pair (c, x) is y_{c,x}, not y_x)."""
    pr = make_tiny_problem(ARCH, n_c=4, n_x=6, seed=10, unaligned=True)
    th = pr.frozen.astype(np.float64)
    data = {"u": pr.u.astype(np.float64), "q": pr.q.astype(np.float64).copy()}
    F = onet.predict(ARCH, th, data)
    perm = np.array([3, 0, 5, 1, 4, 2])
    data2 = {"u": data["u"], "q": data["q"].copy()}
    data2["q"][2] = data["q"][2][perm]
    F2 = onet.predict(ARCH, th, data2)
    np.testing.assert_allclose(F2[2], F[2][perm], rtol=1e-13)
    np.testing.assert_array_equal(np.delete(F2, 2, 0), np.delete(F, 2, 0))


def test_unaligned_sensitivities_shared_points():
    pr = make_tiny_problem(ARCH, n_c=3, n_x=4, seed=11)
    al = {"u": pr.u, "q": pr.q, "v": pr.v}
    un = {"u": pr.u, "q": np.repeat(pr.q[None], 3, 0), "v": pr.v}
    np.testing.assert_allclose(osens.sensitivities(ARCH, pr.frozen, pr.sigma_vi, un),
                               osens.sensitivities(ARCH, pr.frozen, pr.sigma_vi, al), rtol=1e-12)


def test_cfg4u_generator():
    p = make_problem("cfg4u", n_chains=2)
    a = make_problem("cfg4", n_chains=2)
    assert p.u.shape == (1000, 100) and p.q.shape == (1000, 100, 1) and p.v.shape == (1000, 100)
    np.testing.assert_array_equal(p.u, a.u)          # same input functions as cfg4
    assert p.P == a.P and p.k == a.k
    assert np.all((p.q >= 0) & (p.q <= 1))
    assert np.unique(p.q[:, :, 0]).size > 100 * 100   # per-function points
    p2 = make_problem("cfg4u", n_chains=2)
    np.testing.assert_array_equal(p.q, p2.q)
    np.testing.assert_array_equal(p.v, p2.v)
