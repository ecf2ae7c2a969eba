"""Helpers for the -m gpu parity tests: run the CUDA path through the C-ABI binding and compare
with the fp64 oracle under the tolerances of BASELINE.json's north_star."""
import numpy as np

LOGP_RTOL = 1e-5      # north_star: log-posterior within 1e-5 relative
GRAD_RTOL = 1e-5      # north_star: gradient within 1e-5 relative (2-norm and inf-norm, Q26)
STATE_RTOL = 1e-4     # north_star: trajectory end states within 1e-4 relative over L <= 50
# Q26b: the element-wise scale budgets the rounding of tanh' = 1 - y^2 taken from the
# stored fp32 output (2 eta y^2, eta = 4 u: rounding plus the tanh evaluation)
KAPPA_Q26B = 2.0 * 4.0 * 2.0 ** -24 / 1e-5


def torch_cuda():
    import torch
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    return torch


def to_dev(a, dtype):
    torch = torch_cuda()
    return torch.as_tensor(np.ascontiguousarray(a), device="cuda").to(dtype).contiguous()


def gpu_grad(ctx, theta):
    """theta [C x k] float32 -> (logp [C] f64, grad [C x k] f32) through hmc_grad (device ptrs)."""
    torch = torch_cuda()
    from paper_2507_14652_b200 import abi
    th = to_dev(theta, torch.float32)
    C, k = theta.shape
    lp = torch.empty(C, dtype=torch.float64, device="cuda")
    g = torch.empty(C, k, dtype=torch.float32, device="cuda")
    abi.hmc_grad(ctx.ctx, th, lp, g)
    torch.cuda.synchronize()
    return lp.cpu().numpy(), g.cpu().numpy()


def jittered_states(prob, C, scale=0.02, seed=0):
    g = np.random.default_rng(12345 + seed)
    base = prob.frozen[prob.idx].astype(np.float64)
    th = base[None, :] + scale * g.normal(size=(C, prob.k)) * np.maximum(np.abs(base), 0.1)[None, :]
    th[0] = base
    return th.astype(np.float32)


def assert_grad_close(lp, g, lp_ref, g_ref, where=""):
    assert abs(lp - lp_ref) <= LOGP_RTOL * abs(lp_ref), (where, lp, lp_ref, abs(lp - lp_ref) / abs(lp_ref))
    d = g.astype(np.float64) - g_ref
    r2 = np.linalg.norm(d) / np.linalg.norm(g_ref)
    ri = np.max(np.abs(d)) / np.max(np.abs(g_ref))
    assert r2 <= GRAD_RTOL and ri <= GRAD_RTOL, (where, r2, ri)
    return r2, ri


def assert_grad_elementwise(lp, g, lp_ref, g_ref, S, where=""):
    """Q26 at chain-visited states: near a mode ||g|| -> 0, so the bound is per
    entry, scaled by the summation magnitude S_i of that entry (oracle Target.grad_scale with
    kappa = KAPPA_Q26B): |g_i - g_ref_i| <= 1e-5 S_i; log pi within 1e-5 relative."""
    assert abs(lp - lp_ref) <= LOGP_RTOL * abs(lp_ref), (where, lp, lp_ref)
    d = np.abs(g.astype(np.float64) - g_ref)
    worst = np.max(d / np.maximum(S, 1e-300))
    assert worst <= GRAD_RTOL, (where, worst, int(np.argmax(d / np.maximum(S, 1e-300))))
    return worst
