"""Networks F_Theta in fp64: layout, forward, reverse mode.  TEST INFRASTRUCTURE ONLY
(see oracle/__init__.py).

PAPER.md P:68 (F_Theta parameterised by Theta in R^{N_Theta}), P:273 / P:335 (MLPs with
sin / tanh), P:369 + P:527-539 (DeepONet: branch and trunk are feed-forward nets).
DeepONet output F(u, y) = sum_k B_k(u) T_k(y) + b0.
Flat layout: per net, per layer W[out x in] row-major then b[out];
DeepONet b0 last.
Unaligned DeepONet: the query points differ per function, data["q"]
is [n_c, n_x, d_t] and pair (c, x) is F(u_c, y_{c,x}) - the same definition with the
trunk evaluated on every pair's own point (n_c * n_x trunk inputs); the aligned layout
q [n_x, d_t] shares the points across functions (trunk on n_x inputs).
"""
from __future__ import annotations

import numpy as np


def layer_table(arch):
    """[(net, layer, w_off, b_off or None, n_out, n_in, act)] in flat order; plus b0 offset."""
    rows = []
    off = 0
    for ni, net in enumerate(arch.nets):
        for l in range(len(net.widths) - 1):
            n_in, n_out = net.widths[l], net.widths[l + 1]
            w_off = off
            off += n_out * n_in
            b_off = None
            if net.bias[l]:
                b_off = off
                off += n_out
            rows.append((ni, l, w_off, b_off, n_out, n_in, net.acts[l]))
    b0 = None
    if arch.has_b0:
        b0 = off
        off += 1
    return rows, b0, off


def param_count(arch) -> int:
    return layer_table(arch)[2]


def _act(name, z):
    if name == "tanh":
        return np.tanh(z)
    if name == "sin":
        return np.sin(z)
    return z


def _dact(name, z):
    """d act / dz evaluated at the pre-activation z."""
    if name == "tanh":
        t = np.tanh(z)
        return 1.0 - t * t
    if name == "sin":
        return np.cos(z)
    return np.ones_like(z)


def net_forward(arch, theta_full, ni, x):
    """h_0 = x; z_l = h_{l-1} W_l^T + b_l; h_l = act_l(z_l), batched over rows of x.
    Returns (output, [(h_in, z)] per layer) in fp64."""
    rows, _, _ = layer_table(arch)
    h = np.asarray(x, dtype=np.float64)
    tape = []
    for (n_idx, l, w_off, b_off, n_out, n_in, act) in rows:
        if n_idx != ni:
            continue
        W = theta_full[w_off:w_off + n_out * n_in].reshape(n_out, n_in)
        z = h @ W.T
        if b_off is not None:
            z = z + theta_full[b_off:b_off + n_out][None, :]
        tape.append((h, z))
        h = _act(act, z)
    return h, tape


def net_backward(arch, theta_full, ni, tape, dout, grad_full):
    """Reverse mode through net ni given dL/d(output) = dout (rows x n_out).
    Accumulates dL/dW_l = delta_l^T h_{l-1}, dL/db_l = sum_rows delta_l into grad_full."""
    rows, _, _ = layer_table(arch)
    mine = [r for r in rows if r[0] == ni]
    g = np.asarray(dout, dtype=np.float64)
    for li in range(len(mine) - 1, -1, -1):
        (_, l, w_off, b_off, n_out, n_in, act) = mine[li]
        h_in, z = tape[li]
        delta = g * _dact(act, z)
        grad_full[w_off:w_off + n_out * n_in] += (delta.T @ h_in).reshape(-1)
        if b_off is not None:
            grad_full[b_off:b_off + n_out] += delta.sum(axis=0)
        W = theta_full[w_off:w_off + n_out * n_in].reshape(n_out, n_in)
        g = delta @ W
    return g


def _unaligned(data):
    return np.asarray(data["q"]).ndim == 3


def _trunk_inputs(data):
    """Trunk input rows: q [n_x, d_t] (aligned) or q [n_c, n_x, d_t] flattened pair-major."""
    q = np.asarray(data["q"], dtype=np.float64)
    return q.reshape(-1, q.shape[-1]) if q.ndim == 3 else q


def _combine(B, T, data):
    """Sum_k B_ck T_(pair)k for every pair: B T^T (aligned) or row-wise dots (unaligned)."""
    if not _unaligned(data):
        return B @ T.T
    n_c, n_x = np.asarray(data["q"]).shape[:2]
    return np.einsum("ck,cxk->cx", B, T.reshape(n_c, n_x, -1))


def _combine_grads(B, T, E, data):
    """dF-weighted sums: (sum_x E_cx T_(c,x)k  per c,  E_cx B_ck per trunk row)."""
    if not _unaligned(data):
        return E @ T, E.T @ B
    n_c, n_x = E.shape
    T3 = T.reshape(n_c, n_x, -1)
    dB = np.einsum("cx,cxk->ck", E, T3)
    dT = (E[:, :, None] * B[:, None, :]).reshape(n_c * n_x, -1)
    return dB, dT


def predict(arch, theta_full, data):
    """F for every datum: MLP -> [n]; DeepONet -> [n_c, n_x] (each pair (c, x) is
    F(u_c, y_x) = B(u_c) . T(y_x) + b0: branch evaluated once per function, trunk once
    per query point, as the definition reads)."""
    theta_full = np.asarray(theta_full, dtype=np.float64)
    if arch.kind == "mlp":
        out, _ = net_forward(arch, theta_full, 0, data["x"])
        return out[:, 0]
    B, _ = net_forward(arch, theta_full, 0, data["u"])
    T, _ = net_forward(arch, theta_full, 1, _trunk_inputs(data))
    _, b0, _ = layer_table(arch)
    F = _combine(B, T, data)
    if b0 is not None:
        F = F + theta_full[b0]
    return F


def predict_pairwise(arch, theta_full, u_rows, q_rows):
    """DeepONet evaluated pair by pair, F = sum_k B_k(u) T_k(y) + b0 - used by the
    factored == pairwise pin."""
    theta_full = np.asarray(theta_full, dtype=np.float64)
    _, b0, _ = layer_table(arch)
    out = np.empty(len(u_rows))
    for i, (u, q) in enumerate(zip(u_rows, q_rows)):
        B, _ = net_forward(arch, theta_full, 0, np.asarray(u)[None, :])
        T, _ = net_forward(arch, theta_full, 1, np.asarray(q)[None, :])
        s = 0.0
        for kk in range(B.shape[1]):
            s += B[0, kk] * T[0, kk]
        out[i] = s + (theta_full[b0] if b0 is not None else 0.0)
    return out


def loglik_grad(arch, theta_full, data, sigma):
    """Gaussian log-likelihood -sum (y - F)^2 / (2 sigma^2) (Table 5; constants
    dropped, Q7) and its gradient over ALL flat parameters (fp64)."""
    theta_full = np.asarray(theta_full, dtype=np.float64)
    s2 = float(sigma) ** 2
    grad = np.zeros_like(theta_full)
    if arch.kind == "mlp":
        F, tape = net_forward(arch, theta_full, 0, data["x"])
        r = np.asarray(data["y"], dtype=np.float64) - F[:, 0]
        ll = -np.dot(r, r) / (2.0 * s2)
        net_backward(arch, theta_full, 0, tape, (r / s2)[:, None], grad)
        return ll, grad, r
    B, tb = net_forward(arch, theta_full, 0, data["u"])
    T, tt = net_forward(arch, theta_full, 1, _trunk_inputs(data))
    _, b0, _ = layer_table(arch)
    F = _combine(B, T, data)
    if b0 is not None:
        F = F + theta_full[b0]
    R = np.asarray(data["v"], dtype=np.float64) - F
    ll = -np.sum(R * R) / (2.0 * s2)
    E = R / s2                       # d ll / d F
    dB, dT = _combine_grads(B, T, E, data)
    net_backward(arch, theta_full, 0, tb, dB, grad)     # dF/dB_ck = T_(pair)k
    net_backward(arch, theta_full, 1, tt, dT, grad)     # dF/dT_(pair)k = B_ck
    if b0 is not None:
        grad[b0] += E.sum()
    return ll, grad, R


def grad_abs_scale(arch, theta_full, data, sigma, kappa=0.0):
    """Summation scale for element-wise gradient tolerances:
    the same reverse mode run on absolute values, seeded with (|F| + |y|)/sigma^2, so
    S_i >= sum over all product terms of |term| in d ll / d theta_i (the quantity a
    floating-point error bound of the gradient is proportional to).

    kappa > 0 (reading Q26b): the derivative of a tanh unit enters as
    |tanh'(z)| + kappa tanh(z)^2 - the absolute error of tanh' = 1 - y^2 taken from a stored
    output y with relative error eta is 2 eta y^2, so kappa = 2 eta / tol lets the tolerance
    tol * S_i budget it (reverse mode from the layer outputs, as autograd computes tanh')."""
    th = np.abs(np.asarray(theta_full, dtype=np.float64))
    rows, b0, _ = layer_table(arch)
    s2 = float(sigma) ** 2
    S = np.zeros_like(th)

    def fwd(ni, x):
        h = np.asarray(x, dtype=np.float64)
        hs, tape = [], []
        th_signed = np.asarray(theta_full, dtype=np.float64)
        for (n_idx, l, w_off, b_off, n_out, n_in, act) in rows:
            if n_idx != ni:
                continue
            W = th_signed[w_off:w_off + n_out * n_in].reshape(n_out, n_in)
            z = h @ W.T
            if b_off is not None:
                z = z + th_signed[b_off:b_off + n_out][None, :]
            tape.append((h, z))
            h = _act(act, z)
        return h, tape

    def bwd(ni, tape, dout):
        mine = [r for r in rows if r[0] == ni]
        g = dout
        for li in range(len(mine) - 1, -1, -1):
            (_, l, w_off, b_off, n_out, n_in, act) = mine[li]
            h_in, z = tape[li]
            da = np.abs(_dact(act, z))
            if kappa and act == "tanh":
                da = da + kappa * np.tanh(z) ** 2
            delta = g * da
            S[w_off:w_off + n_out * n_in] += (delta.T @ np.abs(h_in)).reshape(-1)
            if b_off is not None:
                S[b_off:b_off + n_out] += delta.sum(axis=0)
            W = th[w_off:w_off + n_out * n_in].reshape(n_out, n_in)
            g = delta @ W

    if arch.kind == "mlp":
        F, tape = fwd(0, data["x"])
        seed = (np.abs(F[:, 0]) + np.abs(np.asarray(data["y"], dtype=np.float64))) / s2
        bwd(0, tape, seed[:, None])
        return S
    B, tb = fwd(0, data["u"])
    T, tt = fwd(1, _trunk_inputs(data))
    F = _combine(B, T, data) + (np.asarray(theta_full, dtype=np.float64)[b0] if b0 is not None else 0.0)
    E = (np.abs(F) + np.abs(np.asarray(data["v"], dtype=np.float64))) / s2
    dB, dT = _combine_grads(np.abs(B), np.abs(T), E, data)
    bwd(0, tb, dB)
    bwd(1, tt, dT)
    if b0 is not None:
        S[b0] += E.sum()
    return S
