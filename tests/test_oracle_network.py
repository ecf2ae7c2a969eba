"""Pins for oracle/network.py and the reduced target (CPU, -m "not gpu").

Each test pins the oracle to something other than itself: numbers printed in the paper,
closed forms, finite differences, invariants (SURVEY §8(c) 'What pins each part')."""
import math
import os

import numpy as np
import pytest

from hmcdata import ArchSpec, NetSpec, make_problem, make_tiny_problem
from hmcdata.generate import n_params
from oracle import hmc as ohmc
from oracle import network as onet

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _arch_from_golden(spec, acts, bias):
    if spec.startswith("deeponet:"):
        br, tr = spec[len("deeponet:"):].split("|")

        def net(s):
            i, rest = s.split("-")
            w, d = rest.split("x")
            widths = [int(i)] + [int(w)] * int(d)
            return NetSpec.plain(widths, hidden=acts)
        return ArchSpec("deeponet", (net(br), net(tr)), has_b0=bool(int(bias)))
    widths = tuple(int(w) for w in spec.split("-"))
    return ArchSpec("mlp", (NetSpec(widths, tuple(acts.split(",")),
                                    tuple(bool(int(b)) for b in bias.split(","))),))


def test_param_counts_printed_in_paper():
    rows = [l.split() for l in open(os.path.join(GOLD, "paper_param_counts.txt"))
            if l.strip() and not l.startswith("#")]
    assert len(rows) == 3
    for name, count, cite, spec, acts, bias in rows:
        arch = _arch_from_golden(spec, acts, bias)
        assert onet.param_count(arch) == int(count), (name, cite)


@pytest.mark.parametrize("name,P,k", [("cfg1", 481, 481), ("cfg2", 12673, 1267),
                                      ("cfg3", 134145, 6707), ("cfg4", 88521, 8852),
                                      ("cfg5", 528641, 20000)])
def test_config_param_counts(name, P, k):
    # hand counts; e.g. 1-20-20-1 = (20+20) + (400+20) + (20+1) = 481
    from hmcdata.configs import CONFIGS
    arch = CONFIGS[name]["arch"]
    assert onet.param_count(arch) == P
    assert n_params(arch) == P   # independent layout walk in the generator


def _case1_arch():
    return ArchSpec("mlp", (NetSpec((1, 2, 1), ("sin", "identity"), (True, False)),))


def test_case1_sine_closed_form():
    """Case I net F = a sin(w1 x + p1) + b sin(w2 x + p2)."""
    arch = _case1_arch()
    # flat order: W1 = (w1, w2), b1 = (p1, p2), W2 = (a, b)
    th = np.array([4.0, -3.0, 0.0, math.pi / 2, 0.4, 0.5])
    assert onet.predict(arch, th, {"x": np.array([[0.0]])})[0] == pytest.approx(0.5, abs=1e-15)
    xs = np.random.default_rng(0).uniform(-2, 2, size=10)
    F = onet.predict(arch, th, {"x": xs[:, None]})
    np.testing.assert_allclose(F, 0.4 * np.sin(4 * xs) + 0.5 * np.sin(-3 * xs + math.pi / 2),
                               rtol=0, atol=1e-14)
    assert np.all(onet.predict(arch, np.zeros(6), {"x": xs[:, None]}) == 0.0)


def test_single_linear_layer():
    """identity, weight 2, bias 1: x = 3 -> 7."""
    arch = ArchSpec("mlp", (NetSpec((1, 1), ("identity",), (True,)),))
    assert onet.predict(arch, np.array([2.0, 1.0]), {"x": np.array([[3.0]])})[0] == 7.0


def test_deeponet_constant_nets():
    """p = 1, branch == 2, trunk == 3, b0 = 0 -> 6 everywhere."""
    # flat: branch W[1x3] (0-2), b (3); trunk W[1x2] (4-5), b (6); b0 (7)
    arch = ArchSpec("deeponet", (NetSpec((3, 1), ("identity",), (True,)),
                                 NetSpec((2, 1), ("identity",), (True,))), has_b0=True)
    th = np.zeros(onet.param_count(arch))
    th[3] = 2.0
    th[6] = 3.0
    g = np.random.default_rng(1)
    data = {"u": g.normal(size=(4, 3)), "q": g.normal(size=(5, 2))}
    np.testing.assert_array_equal(onet.predict(arch, th, data), np.full((4, 5), 6.0))


def test_deeponet_factored_equals_pairwise_and_bilinear():
    arch = ArchSpec("deeponet", (NetSpec.plain((4, 7, 5)), NetSpec.plain((2, 6, 5), last="tanh")),
                    has_b0=True)
    pr = make_tiny_problem(arch, n_c=6, n_x=9, seed=3)
    th = pr.frozen.astype(np.float64)
    data = {"u": pr.u.astype(np.float64), "q": pr.q.astype(np.float64)}
    F = onet.predict(arch, th, data)
    cc, xx = np.meshgrid(np.arange(6), np.arange(9), indexing="ij")
    Fp = onet.predict_pairwise(arch, th, data["u"][cc.ravel()], data["q"][xx.ravel()])
    np.testing.assert_allclose(F.ravel(), Fp, rtol=1e-13, atol=1e-13)
    # bilinearity: scale branch last layer (W and b) by alpha
    rows, b0, _ = onet.layer_table(arch)
    last_branch = [r for r in rows if r[0] == 0][-1]
    _, _, w_off, b_off, n_out, n_in, _ = last_branch
    th2 = th.copy()
    th2[w_off:w_off + n_out * n_in] *= 2.5
    th2[b_off:b_off + n_out] *= 2.5
    F2 = onet.predict(arch, th2, data)
    np.testing.assert_allclose(F2 - th[b0], 2.5 * (F - th[b0]), rtol=1e-12, atol=1e-12)


def _fd_check(prob, n_coords=12, seed=0):
    tgt = ohmc.Target(prob)
    g = np.random.default_rng(seed)
    th = prob.frozen[prob.idx].astype(np.float64) + 0.05 * g.normal(size=prob.k)
    lp, grad = tgt.logp_grad(th)
    h = 1e-6
    coords = g.choice(prob.k, size=min(n_coords, prob.k), replace=False)
    for j in coords:
        e = np.zeros(prob.k)
        e[j] = h
        fd = (tgt.logp_grad(th + e)[0] - tgt.logp_grad(th - e)[0]) / (2 * h)
        scale = max(abs(grad[j]), 1e-3 * np.max(np.abs(grad)))
        assert abs(fd - grad[j]) / scale < 1e-5, (j, fd, grad[j])


def test_fd_gradient_mlp_tanh():
    arch = ArchSpec("mlp", (NetSpec.plain((3, 9, 7, 1)),))
    _fd_check(make_tiny_problem(arch, n=37, active_frac=0.6, seed=1, noise=0.5))


def test_fd_gradient_mlp_sin_no_bias():
    arch = ArchSpec("mlp", (NetSpec((2, 5, 4, 1), ("sin", "tanh", "identity"), (True, False, False)),))
    _fd_check(make_tiny_problem(arch, n=23, active_frac=1.0, seed=2, noise=0.5))


def test_fd_gradient_case1():
    _fd_check(make_tiny_problem(_case1_arch(), n=20, seed=4, noise=1e-1))


def test_fd_gradient_deeponet():
    arch = ArchSpec("deeponet", (NetSpec.plain((4, 6, 5)), NetSpec.plain((2, 6, 5), last="tanh")),
                    has_b0=True)
    _fd_check(make_tiny_problem(arch, n_c=7, n_x=11, active_frac=0.7, seed=5, noise=0.5), n_coords=20)


def test_linear_model_gradient_closed_form():
    """F = x.w + b: d ll/dw = X^T r / s^2, d ll/db = sum r / s^2."""
    arch = ArchSpec("mlp", (NetSpec((4, 1), ("identity",), (True,)),))
    g = np.random.default_rng(7)
    X, y, th = g.normal(size=(30, 4)), g.normal(size=30), g.normal(size=5)
    ll, grad, r = onet.loglik_grad(arch, th, {"x": X, "y": y}, 0.3)
    res = y - X @ th[:4] - th[4]
    assert ll == pytest.approx(-np.dot(res, res) / (2 * 0.09), rel=1e-14)
    np.testing.assert_allclose(grad[:4], X.T @ res / 0.09, rtol=1e-12)
    assert grad[4] == pytest.approx(res.sum() / 0.09, rel=1e-12)


def test_gradient_linear_over_data():
    """gradient of a sum of per-datum terms = sum of per-datum gradients."""
    arch = ArchSpec("mlp", (NetSpec.plain((2, 6, 1)),))
    pr = make_tiny_problem(arch, n=9, seed=8)
    th = pr.frozen.astype(np.float64)
    X, y = pr.x.astype(np.float64), pr.y.astype(np.float64)
    _, gall, _ = onet.loglik_grad(arch, th, {"x": X, "y": y}, 0.2)
    gs = sum(onet.loglik_grad(arch, th, {"x": X[i:i + 1], "y": y[i:i + 1]}, 0.2)[1] for i in range(9))
    np.testing.assert_allclose(gall, gs, rtol=1e-12, atol=1e-12)


def test_masked_gradient_equals_full_coordinates():
    """Reduced-target gradient = full-target gradient at the assembled point, restricted
    to idx (chain rule with frozen coordinates)."""
    arch = ArchSpec("mlp", (NetSpec.plain((2, 8, 1)),))
    pr = make_tiny_problem(arch, n=15, active_frac=0.4, seed=9)
    full = make_tiny_problem(arch, n=15, active_frac=1.0, seed=9)
    t_red, t_full = ohmc.Target(pr), ohmc.Target(full)
    th_full = full.frozen.astype(np.float64) + 0.1
    lp_f, g_f = t_full.logp_grad(th_full)
    # reduced target with frozen = th_full (so the assembled point is the same)
    pr.frozen = th_full.astype(np.float64)
    t_red = ohmc.Target(pr)
    lp_r, g_r = t_red.logp_grad(th_full[pr.idx])
    # priors differ only by frozen-coordinate terms (constant in theta_s)
    frozen_mask = np.ones(full.P, bool)
    frozen_mask[pr.idx] = False
    assert lp_r - lp_f == pytest.approx(np.sum(th_full[frozen_mask] ** 2) / 2.0, rel=1e-12)
    np.testing.assert_allclose(g_r, g_f[pr.idx], rtol=1e-13, atol=1e-13)


def test_zero_data_prior_peak():
    """zero data, prior N(0,1), theta = 0 -> normalised log density -(D/2) log 2 pi;
    gradient of -|theta|^2/2 is -theta."""
    arch = ArchSpec("mlp", (NetSpec.plain((2, 3, 1)),))
    pr = make_tiny_problem(arch, n=0, seed=10, prior=1.0)
    t = ohmc.Target(pr)
    lp, g = t.logp_grad(np.zeros(pr.k))
    assert lp + t.logpost_const() == pytest.approx(-(pr.k / 2) * math.log(2 * math.pi), rel=1e-14)
    th = np.random.default_rng(0).normal(size=pr.k)
    lp, g = t.logp_grad(th)
    np.testing.assert_allclose(g, -th, rtol=1e-15)
    assert lp == pytest.approx(-0.5 * np.dot(th, th), rel=1e-15)


def test_conjugate_one_parameter_quadratic():
    """F = w x: log p(w) = -a w^2/2 + b w - c with a = sum x^2/s^2 + 1/sp^2,
    b = sum x y / s^2, c = sum y^2/(2 s^2) (hand-derived)."""
    arch = ArchSpec("mlp", (NetSpec((1, 1), ("identity",), (False,)),))
    pr = make_tiny_problem(arch, n=25, seed=11, noise=0.4, prior=2.0)
    t = ohmc.Target(pr)
    x, y = pr.x[:, 0].astype(np.float64), pr.y.astype(np.float64)
    a = np.dot(x, x) / 0.16 + 1 / 4.0
    b = np.dot(x, y) / 0.16
    c = np.dot(y, y) / 0.32
    for w in (-1.3, 0.0, 0.7):
        lp, g = t.logp_grad(np.array([w]))
        assert lp == pytest.approx(-0.5 * a * w * w + b * w - c, rel=1e-13)
        assert g[0] == pytest.approx(-a * w + b, rel=1e-12, abs=1e-12)


def test_grad_scale_bounds_gradient():
    """S_i >= |g_i| (the scale sums absolute values of the gradient's terms)."""
    arch = ArchSpec("deeponet", (NetSpec.plain((3, 5, 4)), NetSpec.plain((2, 5, 4), last="tanh")),
                    has_b0=True)
    pr = make_tiny_problem(arch, n_c=5, n_x=6, seed=12, active_frac=0.8)
    t = ohmc.Target(pr)
    th = pr.frozen[pr.idx].astype(np.float64)
    _, g = t.logp_grad(th)
    S = t.grad_scale(th)
    assert np.all(S >= np.abs(g) * (1 - 1e-12))


def test_config_generators_deterministic_and_shaped():
    p1 = make_problem("cfg2")
    p2 = make_problem("cfg2")
    np.testing.assert_array_equal(p1.x, p2.x)
    np.testing.assert_array_equal(p1.idx, p2.idx)
    assert p1.k == 1267 and np.all(np.diff(p1.idx) > 0)
    p5 = make_problem("cfg5")
    assert p5.u.shape == (512, 5) and p5.q.shape == (2048, 2) and p5.v.shape == (512, 2048)
    assert p5.k == 20000
    p4 = make_problem("cfg4")
    assert p4.u.shape == (1000, 100) and p4.q.shape == (100, 1) and p4.v.shape == (1000, 100)


KAPPA_Q26B = 2.0 * 4.0 * 2.0 ** -24 / 1e-5   # 2 eta / tol, eta = 4 u (Q26b)


def test_grad_scale_kappa_no_effect_without_tanh():
    pr = make_problem("blr", n_chains=1)
    t = ohmc.Target(pr)
    th = np.array([0.3, -1.0, 0.5, 2.0])
    np.testing.assert_array_equal(t.grad_scale(th), t.grad_scale(th, KAPPA_Q26B))


def test_grad_scale_kappa_budgets_output_derivative_rounding(monkeypatch):
    """Q26b pin: reverse mode that takes tanh' = 1 - y^2 from the fp32-ROUNDED layer output y
    (autograd's arithmetic; everything else exact) perturbs each unit's derivative by up to
    2 u y^2.  At strongly saturated units that breaks |dg_i| <= 1e-5 S_i (kappa = 0) but stays
    within 1e-5 S_i(kappa) - the first-order bound of that perturbation."""
    from oracle import network as onet
    arch = ArchSpec("mlp", (NetSpec.plain((2, 16, 16, 1)),))
    pr = make_tiny_problem(arch, n=200, seed=13, active_frac=1.0)
    t = ohmc.Target(pr)
    th = 2.5 * pr.frozen[pr.idx].astype(np.float64) / max(np.std(pr.frozen), 1e-12)   # saturating weights
    _, g_ref = t.logp_grad(th)
    exact = onet._dact

    def dact_from_fp32_output(name, z):
        if name == "tanh":
            y = np.tanh(z).astype(np.float32).astype(np.float64)
            return 1.0 - y * y
        return exact(name, z)

    monkeypatch.setattr(onet, "_dact", dact_from_fp32_output)
    _, g_out = t.logp_grad(th)
    monkeypatch.setattr(onet, "_dact", exact)
    d = np.abs(g_out - g_ref)
    assert np.max(d / t.grad_scale(th)) > 1e-5                 # the mechanism is exercised
    assert np.max(d / t.grad_scale(th, KAPPA_Q26B)) <= 1e-5


def test_config_json_files():
    """configs/cfg{1..5}.json: every BASELINE config, its unstated fields listed under
    "assumed" with the reading, and the generator's parameter / mask sizes from them."""
    import json
    import os
    from hmcdata.configs import CONFIG_DIR, load_config
    want = {"cfg1": (481, 481), "cfg2": (12673, 1267), "cfg3": (134145, 6707), "cfg4": (88521, 8852),
            "cfg5": (528641, 20000)}
    for name, (P, k) in want.items():
        d = json.load(open(os.path.join(CONFIG_DIR, name + ".json")))
        assert d["name"] == name and "assumed" in d and "seed" in d["assumed"]
        if name != "cfg1":
            assert "prior_sigma" in d["assumed"] and "mask" in d["assumed"]
        assert load_config(name)["cid"] == int(name[-1])
        p = make_problem(name, n_chains=1)
        assert (p.P, p.k) == (P, k)
