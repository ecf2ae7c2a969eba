"""Thin ctypes binding of libhmc.so (include/hmc.h).  Argument marshalling only: every step of
the hot path runs in the library's CUDA kernels.  There is no CPU fallback - if the library is
missing or fails to load, every call raises.

Arrays may be torch tensors (device or host, contiguous, matching dtype) or NumPy arrays (host).
The functions keep the C names: hmc_setup, hmc_grad, hmc_trajectory, hmc_sample, ...
"""
from __future__ import annotations

import ctypes
import os
from typing import Optional

import numpy as np

HMC_OK, HMC_E_CONFIG, HMC_E_CUDA, HMC_E_NCCL, HMC_E_OOM, HMC_E_STATE = 0, 1, 3, 4, 5, 6
HMC_MLP, HMC_DEEPONET = 0, 1
ACT = {"identity": 0, "tanh": 1, "sin": 2}
MODE = {"single": 0, "data": 1, "chain": 2}
SHARD = {"rows": 0, "points_xb": 1, "points_xc": 2}

LIB_PATH = os.environ.get("HMC_LIB") or os.path.join(os.path.dirname(os.path.abspath(__file__)), "libhmc.so")


class HmcError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"libhmc status {code}: {msg}")
        self.code = code


class hmc_net(ctypes.Structure):
    _fields_ = [("n_layers", ctypes.c_int32), ("widths", ctypes.POINTER(ctypes.c_int32)),
                ("acts", ctypes.POINTER(ctypes.c_int32)), ("has_bias", ctypes.POINTER(ctypes.c_int32))]


class hmc_arch(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_int32), ("net", hmc_net * 2), ("has_b0", ctypes.c_int32)]


class hmc_data(ctypes.Structure):
    _fields_ = [("x", ctypes.c_void_p), ("y", ctypes.c_void_p), ("n", ctypes.c_int64),
                ("u", ctypes.c_void_p), ("q", ctypes.c_void_p), ("v", ctypes.c_void_p),
                ("n_c", ctypes.c_int64), ("n_x", ctypes.c_int64), ("n_global", ctypes.c_int64),
                ("q_per_pair", ctypes.c_int32)]


class hmc_config(ctypes.Structure):
    _fields_ = [("frozen", ctypes.c_void_p), ("idx", ctypes.c_void_p), ("P", ctypes.c_int64),
                ("k", ctypes.c_int64), ("noise_sigma", ctypes.c_double),
                ("prior_sigma", ctypes.c_double), ("inv_mass", ctypes.c_void_p),
                ("seed", ctypes.c_uint64), ("n_chains", ctypes.c_int32),
                ("chain_ids", ctypes.c_void_p), ("mode", ctypes.c_int32), ("rank", ctypes.c_int32),
                ("world", ctypes.c_int32), ("shard", ctypes.c_int32), ("nccl_id", ctypes.c_void_p),
                ("exchange", ctypes.c_int32)]


EXPORTS = ["hmc_comm_unique_id", "hmc_setup", "hmc_grad", "hmc_logpost_const", "hmc_trajectory",
           "hmc_sample", "hmc_destroy", "hmc_last_error", "hmc_launch_counts", "hmc_philox_words",
           "hmc_momentum", "hmc_engine_info", "hmc_profile", "hmc_profile_read", "hmc_debug_gemm",
           "hmc_debug_tc_profile", "hmc_debug_tc_timeline", "hmc_sensitivity", "hmc_adapt", "hmc_predict",
           "hmc_diagnostics", "hmc_partition", "hmc_divergences", "hmc_debug_set_engine",
           "hmc_debug_data_phase", "hmc_debug_xb_permute", "hmc_debug_nw_profile"]


class hmc_prof_rec(ctypes.Structure):
    _fields_ = [("name", ctypes.c_char * 64), ("ms", ctypes.c_double), ("flops", ctypes.c_double),
                ("bytes", ctypes.c_double), ("step", ctypes.c_int32)]

_lib = None


def lib():
    """Load libhmc.so (in-tree build).  Raises if it is missing: no fallback exists."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(f"{LIB_PATH} is not built; run `make` or __graft_entry__.build()")
    # libhmc.so needs libnccl.so.2.  Load torch first so its bundled NCCL (the one libtorch_cuda
    # was built against) is the copy in the process; loading the system NCCL first would leave
    # torch with unresolved NCCL symbols.
    import torch  # noqa: F401  (plumbing: device memory, streams, process groups)
    L = ctypes.CDLL(LIB_PATH)
    vp, i32, i64, u32, u64, dbl = (ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_uint32,
                                   ctypes.c_uint64, ctypes.c_double)
    L.hmc_comm_unique_id.argtypes = [vp]
    L.hmc_setup.argtypes = [ctypes.POINTER(hmc_arch), ctypes.POINTER(hmc_data),
                            ctypes.POINTER(hmc_config), vp, ctypes.POINTER(vp)]
    L.hmc_grad.argtypes = [vp, vp, vp, vp, vp]
    L.hmc_logpost_const.argtypes = [vp, ctypes.POINTER(dbl)]
    L.hmc_trajectory.argtypes = [vp, vp, vp, vp, dbl, i32, i64, vp, vp, vp]
    L.hmc_sample.argtypes = [vp, vp, vp, vp, dbl, i32, i64, i32, vp, vp, vp, vp]
    L.hmc_destroy.argtypes = [vp]
    L.hmc_last_error.argtypes = [vp]
    L.hmc_last_error.restype = ctypes.c_char_p
    L.hmc_launch_counts.argtypes = [vp, ctypes.POINTER(i64), ctypes.POINTER(i64), ctypes.POINTER(i64)]
    L.hmc_philox_words.argtypes = [u64, u32, u32, u32, i64, vp, vp]
    L.hmc_momentum.argtypes = [vp, i64, vp, vp]
    L.hmc_engine_info.argtypes = [vp]
    L.hmc_engine_info.restype = ctypes.c_char_p
    L.hmc_profile.argtypes = [vp, i32]
    L.hmc_debug_gemm.argtypes = [i32, i32, i32, i32, i32, i32, i32, vp, i64, i64, vp, i64, i64, vp, i64,
                                 i64, vp]
    L.hmc_profile_read.argtypes = [vp, i32, ctypes.POINTER(hmc_prof_rec), ctypes.POINTER(i32)]
    for name in EXPORTS:
        if name not in ("hmc_last_error", "hmc_engine_info"):
            getattr(L, name).restype = ctypes.c_int
    _lib = L
    return L


_TORCH_DT = {np.dtype(np.float32): "torch.float32", np.dtype(np.float64): "torch.float64",
             np.dtype(np.uint8): "torch.uint8", np.dtype(np.int32): "torch.int32",
             np.dtype(np.uint32): "torch.uint32"}

# (C, k) of the contexts created through this module, for the shape checks of _arg
_CTX_SHAPE: dict = {}


def _ptr(a, keep: list, dtype=None):
    """Raw pointer of an INPUT torch tensor or NumPy array (None -> NULL).  A NumPy input of
    another dtype or layout is converted (a copy the library only reads); a torch tensor must
    already have the dtype and be contiguous."""
    return _arg(a, keep, dtype, out=False)


def _arg(a, keep: list, dtype=None, count=None, out=True, name="array"):
    """Raw pointer of an argument the library reads (out=False) or WRITES (out=True).  Written
    arguments are never copied: a NumPy array or torch tensor of the wrong dtype, a
    non-contiguous one, or one with the wrong element count raises (the library would otherwise
    write past its end, or into a temporary copy the caller never sees)."""
    if a is None:
        return None
    if hasattr(a, "data_ptr"):          # torch.Tensor
        if dtype is not None and str(a.dtype) != _TORCH_DT[np.dtype(dtype)]:
            raise TypeError(f"{name}: torch dtype {a.dtype}, expected {_TORCH_DT[np.dtype(dtype)]}")
        if not a.is_contiguous():
            raise ValueError(f"{name}: tensor must be contiguous")
        if count is not None and a.numel() != count:
            raise ValueError(f"{name}: {a.numel()} elements, expected {count}")
        keep.append(a)
        return a.data_ptr()
    if out:
        if not isinstance(a, np.ndarray):
            raise TypeError(f"{name}: output arguments must be NumPy arrays or torch tensors")
        if dtype is not None and a.dtype != np.dtype(dtype):
            raise TypeError(f"{name}: dtype {a.dtype}, expected {np.dtype(dtype)}")
        if not a.flags.c_contiguous or not a.flags.writeable:
            raise ValueError(f"{name}: output array must be C-contiguous and writeable")
        arr = a
    else:
        arr = np.ascontiguousarray(a, dtype=dtype) if dtype is not None else np.ascontiguousarray(a)
    if count is not None and arr.size != count:
        raise ValueError(f"{name}: {arr.size} elements, expected {count}")
    keep.append(arr)
    return arr.ctypes.data


def _shape(ctx):
    """(C, k) of a context made by this module (None, None for a foreign handle)."""
    return _CTX_SHAPE.get(ctx, (None, None))


def _n(*dims):
    return None if any(d is None for d in dims) else int(np.prod(dims))


def _check(rc, ctx=None):
    if rc != HMC_OK:
        msg = lib().hmc_last_error(ctx)
        raise HmcError(rc, msg.decode() if msg else "")


def _stream(stream):
    if stream is None:
        return None
    if hasattr(stream, "cuda_stream"):
        return stream.cuda_stream
    return int(stream)


def hmc_comm_unique_id() -> bytes:
    buf = (ctypes.c_uint8 * 128)()
    _check(lib().hmc_comm_unique_id(buf))
    return bytes(buf)


def make_arch(kind: str, nets, has_b0: bool, keep: list) -> hmc_arch:
    """nets: sequence of (widths, acts, has_bias) python sequences."""
    a = hmc_arch()
    a.kind = HMC_MLP if kind == "mlp" else HMC_DEEPONET
    for i, (widths, acts, bias) in enumerate(nets):
        w = (ctypes.c_int32 * len(widths))(*widths)
        ac = (ctypes.c_int32 * len(acts))(*[ACT[x] if isinstance(x, str) else int(x) for x in acts])
        b = (ctypes.c_int32 * len(bias))(*[int(bool(x)) for x in bias])
        keep += [w, ac, b]
        a.net[i] = hmc_net(len(widths) - 1, w, ac, b)
    a.has_b0 = int(bool(has_b0))
    return a


def hmc_setup(arch: hmc_arch, data: hmc_data, cfg: hmc_config, stream=None) -> int:
    ctx = ctypes.c_void_p()
    _check(lib().hmc_setup(ctypes.byref(arch), ctypes.byref(data), ctypes.byref(cfg),
                           _stream(stream), ctypes.byref(ctx)))
    return ctx.value


def hmc_grad(ctx, theta, logp, grad, stream=None):
    keep = []
    C, k = _shape(ctx)
    _check(lib().hmc_grad(ctx, _arg(theta, keep, np.float32, _n(C, k), out=False, name="theta"),
                          _arg(logp, keep, np.float64, C, name="logp"),
                          _arg(grad, keep, np.float32, _n(C, k), name="grad"), _stream(stream)), ctx)


def hmc_logpost_const(ctx) -> float:
    c = ctypes.c_double()
    _check(lib().hmc_logpost_const(ctx, ctypes.byref(c)), ctx)
    return c.value


def _state_args(ctx, theta, logp, grad, keep):
    """theta [C x k] f32, logp [C] f64, grad [C x k] f32: in/out chain state (never copied)."""
    C, k = _shape(ctx)
    return (_arg(theta, keep, np.float32, _n(C, k), name="theta"), _arg(logp, keep, np.float64, C, name="logp"),
            _arg(grad, keep, np.float32, _n(C, k), name="grad"))


def hmc_trajectory(ctx, theta, logp, grad, eps, L, it, acc=None, dH=None, stream=None):
    keep = []
    C, _ = _shape(ctx)
    th, lp, g = _state_args(ctx, theta, logp, grad, keep)
    _check(lib().hmc_trajectory(ctx, th, lp, g, float(eps), int(L), int(it),
                                _arg(acc, keep, np.uint8, C, name="acc"),
                                _arg(dH, keep, np.float64, C, name="dH"), _stream(stream)), ctx)


def hmc_sample(ctx, theta, logp, grad, eps, L, iter0, S, samples, acc=None, dH=None, stream=None):
    keep = []
    C, k = _shape(ctx)
    th, lp, g = _state_args(ctx, theta, logp, grad, keep)
    _check(lib().hmc_sample(ctx, th, lp, g, float(eps), int(L), int(iter0), int(S),
                            _arg(samples, keep, np.float32, _n(C, S, k), name="samples"),
                            _arg(acc, keep, np.uint8, _n(C, S), name="acc"),
                            _arg(dH, keep, np.float64, _n(C, S), name="dH"), _stream(stream)), ctx)


def hmc_destroy(ctx):
    if ctx:
        _check(lib().hmc_destroy(ctx))


def hmc_launch_counts(ctx):
    a, b, c = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64()
    _check(lib().hmc_launch_counts(ctx, ctypes.byref(a), ctypes.byref(b), ctypes.byref(c)), ctx)
    return a.value, b.value, c.value


def hmc_philox_words(seed, tag, it, chain, nblocks, out, stream=None):
    keep = []
    _check(lib().hmc_philox_words(int(seed), int(tag), int(it), int(chain), int(nblocks),
                                  _ptr(out, keep), _stream(stream)))


def hmc_momentum(ctx, it, out, stream=None):
    keep = []
    C, k = _shape(ctx)
    _check(lib().hmc_momentum(ctx, int(it), _arg(out, keep, np.float32, _n(C, k), name="p"), _stream(stream)), ctx)


def hmc_divergences(ctx, reset: bool = False):
    """Per-chain counts of divergent trajectories (non-finite or |dH| > 1000) since creation or the
    last reset (include/hmc.h hmc_divergences); a uint32 NumPy array [C]."""
    C, _ = _shape(ctx)
    if C is None:
        raise ValueError("hmc_divergences needs a context created through abi.Context")
    out = np.zeros(C, dtype=np.uint32)
    L = lib()
    L.hmc_divergences.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int32]
    _check(L.hmc_divergences(ctx, out.ctypes.data, int(bool(reset))), ctx)
    return out


def hmc_debug_data_phase(ctx, phase, inp=None, inp2=None, out=None, out2=None):
    """Test hook (include/hmc.h): one phase of a DATA-mode evaluation on an exchange='emulated'
    context; device tensors."""
    keep = []
    L = lib()
    L.hmc_debug_data_phase.argtypes = [ctypes.c_void_p, ctypes.c_int32] + [ctypes.c_void_p] * 5
    _check(L.hmc_debug_data_phase(ctx, int(phase), _ptr(inp, keep), _ptr(inp2, keep), _ptr(out, keep),
                                  _ptr(out2, keep), None), ctx)


def hmc_debug_xb_permute(direction, C, G, n_loc, p, inp, out):
    """Test hook: k_xb_gather (direction 0) or k_xb_scatter (1) on device tensors."""
    keep = []
    L = lib()
    L.hmc_debug_xb_permute.argtypes = [ctypes.c_int32] * 3 + [ctypes.c_int64, ctypes.c_int32] + [ctypes.c_void_p] * 3
    _check(L.hmc_debug_xb_permute(int(direction), int(C), int(G), int(n_loc), int(p), _ptr(inp, keep),
                                  _ptr(out, keep), None))


def hmc_debug_set_engine(mode: int):
    """Test hook: 1 = contexts set up afterwards run every GEMM on the SIMT engine; 0 = automatic."""
    L = lib()
    L.hmc_debug_set_engine.argtypes = [ctypes.c_int32]
    _check(L.hmc_debug_set_engine(int(mode)))


def hmc_engine_info(ctx) -> str:
    return lib().hmc_engine_info(ctx).decode()


def hmc_debug_gemm(engine, a_kmajor, b_kmajor, M, N, K, batch, A, lda, sA, B, ldb, sB, C, ldc, sC,
                   stream=None):
    keep = []
    _check(lib().hmc_debug_gemm(int(engine), int(a_kmajor), int(b_kmajor), M, N, K, batch,
                                _ptr(A, keep), lda, sA, _ptr(B, keep), ldb, sB, _ptr(C, keep), ldc, sC,
                                _stream(stream)))


TC_PROF_SLOTS = ["tmaA_wait_slot", "mma_wait_acc", "mma_wait_operands", "conv_wait_A", "conv_wait_aslot",
                 "epi_wait_acc", "epi_wait_prefetch", "epi_output", "kernel_cycles", "conv_wait_B", "tmaB_wait_slot",
                 "mma_issue"]


def hmc_debug_tc_profile(reset: bool = False):
    """Per-role barrier wait cycles of the tcgen05 engine (HMC_TC_PROF=1), summed over CTAs."""
    out = (ctypes.c_uint64 * 256)()
    L = lib()
    L.hmc_debug_tc_profile.argtypes = [ctypes.c_void_p, ctypes.c_int32]
    _check(L.hmc_debug_tc_profile(out, int(bool(reset))))
    v = list(out)
    return {vid: dict(zip(TC_PROF_SLOTS, v[16 * vid:16 * vid + len(TC_PROF_SLOTS)])) for vid in range(16)
            if any(v[16 * vid:16 * vid + 16])}


def hmc_debug_tc_timeline():
    """CTA-0 timeline [24 x 256] (clock64) of the last tcgen05 GEMM with HMC_TC_PROF=2."""
    out = (ctypes.c_uint64 * (24 * 256))()
    L = lib()
    L.hmc_debug_tc_timeline.argtypes = [ctypes.c_void_p]
    _check(L.hmc_debug_tc_timeline(out))
    return np.array(list(out), dtype=np.int64).reshape(24, 256)


def hmc_profile(ctx, enable: bool):
    _check(lib().hmc_profile(ctx, int(bool(enable))), ctx)


def hmc_profile_read(ctx):
    """[(name, ms, flops, bytes, step)] of the last replayed trajectory."""
    n = ctypes.c_int32()
    _check(lib().hmc_profile_read(ctx, 0, None, ctypes.byref(n)), ctx)
    recs = (hmc_prof_rec * max(n.value, 1))()
    _check(lib().hmc_profile_read(ctx, n.value, recs, ctypes.byref(n)), ctx)
    return [(r.name.decode(), r.ms, r.flops, r.bytes, r.step) for r in recs[:n.value]]


def hmc_adapt(ctx, theta, logp, grad, eps0, L, iter0, n_adapt, delta, acc=None, dH=None, stream=None):
    """Dual-averaging warm-up (include/hmc.h hmc_adapt); returns the per-chain eps_bar (NumPy)."""
    keep = []
    L_ = lib()
    L_.hmc_adapt.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_double,
                             ctypes.c_int32, ctypes.c_int64, ctypes.c_int32, ctypes.c_double, ctypes.c_void_p,
                             ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]
    C = int(theta.shape[0])
    out = np.empty(C, dtype=np.float64)
    th, lp, g = _state_args(ctx, theta, logp, grad, keep)
    _check(L_.hmc_adapt(ctx, th, lp, g, float(eps0), int(L), int(iter0), int(n_adapt), float(delta), out.ctypes.data,
                        _arg(acc, keep, np.uint8, C * int(n_adapt), name="acc"),
                        _arg(dH, keep, np.float64, C * int(n_adapt), name="dH"), _stream(stream)), ctx)
    return out


def hmc_predict(ctx, samples, stream=None):
    """Posterior predictive mean / variance over the inputs of `ctx` (a Context); samples [S x k]."""
    keep = []
    L = lib()
    L.hmc_predict.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p,
                              ctypes.c_void_p]
    S = int(samples.shape[0])
    N = int(getattr(ctx, "_n_out", 0))
    mean = np.empty(N, dtype=np.float64)
    var = np.empty(N, dtype=np.float64)
    _check(L.hmc_predict(ctx.ctx, _ptr(samples, keep, np.float32), S, mean.ctypes.data, var.ctypes.data,
                         _stream(stream)), ctx.ctx)
    return mean, var


def hmc_diagnostics(samples, stream=None):
    """split-R^ and ESS per parameter of samples [C x S x k] (include/hmc.h hmc_diagnostics)."""
    keep = []
    L = lib()
    L.hmc_diagnostics.argtypes = [ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_int64,
                                  ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]
    C, S, k = (int(v) for v in samples.shape)
    rhat = np.empty(k, dtype=np.float64)
    ess = np.empty(k, dtype=np.float64)
    _check(L.hmc_diagnostics(_ptr(samples, keep, np.float32), C, S, k, rhat.ctypes.data, ess.ctypes.data,
                             _stream(stream)))
    return rhat, ess


def hmc_partition(s2, tau: float, rule: str = "ge", stream=None):
    """Theta_s of eqn:threshold on the GPU: the N^ most sensitive flat indices (ascending int32
    NumPy array) for sensitivities s2 [P] (NumPy or torch, fp64), rule "ge" (text) or "le"."""
    keep = []
    arr = s2 if hasattr(s2, "data_ptr") else np.ascontiguousarray(s2, dtype=np.float64)
    P = int(arr.shape[0])
    out = np.empty(P, dtype=np.int32)
    nh = ctypes.c_int64(0)
    L = lib()
    L.hmc_partition.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_double, ctypes.c_int32,
                                ctypes.c_void_p, ctypes.POINTER(ctypes.c_int64), ctypes.c_void_p]
    _check(L.hmc_partition(_ptr(arr, keep), P, float(tau), 0 if rule == "ge" else 1, out.ctypes.data,
                           ctypes.byref(nh), _stream(stream)))
    return out[:nh.value].copy()


def hmc_sensitivity(problem, mu=None, sigma_vi=None, stream=None):
    """S_i^2 for every flat parameter (eqn:sensitivities) of problem.arch on problem's data, at
    mu (default problem.frozen) with VI sds sigma_vi (default problem.sigma_vi).  Returns a
    float64 NumPy array [P]."""
    keep = []
    arch = problem.arch
    a = make_arch(arch.kind, [(n.widths, n.acts, n.bias) for n in arch.nets], arch.has_b0, keep)
    d = hmc_data()
    if arch.kind == "mlp":
        d.x = _ptr(problem.x, keep, np.float32)
        d.y = _ptr(problem.y, keep, np.float32)
        d.n = int(problem.x.shape[0])
    else:
        d.u = _ptr(problem.u, keep, np.float32)
        d.q = _ptr(problem.q, keep, np.float32)
        d.v = _ptr(problem.v, keep, np.float32)
        d.n_c, d.n_x = int(problem.u.shape[0]), int(problem.v.shape[1])
        d.q_per_pair = int(len(problem.q.shape) == 3)  # unaligned: q [n_c, n_x, d_t]
    mu = problem.frozen if mu is None else mu
    sigma_vi = problem.sigma_vi if sigma_vi is None else sigma_vi
    P = int(np.asarray(mu).shape[0]) if not hasattr(mu, "device") else int(mu.shape[0])
    out = np.empty(P, dtype=np.float64)
    L = lib()
    L.hmc_sensitivity.argtypes = [ctypes.POINTER(hmc_arch), ctypes.POINTER(hmc_data), ctypes.c_void_p,
                                  ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]
    _check(L.hmc_sensitivity(ctypes.byref(a), ctypes.byref(d), _ptr(mu, keep, np.float32),
                             _ptr(sigma_vi, keep, np.float32), out.ctypes.data, _stream(stream)))
    return out


class Context:
    """Owns one libhmc context built from a problem description (any object with the fields of
    hmcdata.Problem: arch, x/y or u/q/v, frozen, idx, noise_sigma, prior_sigma, inv_mass, seed,
    n_chains, chain_ids).  Marshalling only."""

    def __init__(self, problem, mode: str = "single", rank: int = 0, world: int = 1,
                 nccl_id: Optional[bytes] = None, n_global: int = 0, chain_ids=None,
                 n_chains: Optional[int] = None, shard: str = "rows", exchange: str = "nccl"):
        keep = []
        arch = problem.arch
        nets = [(n.widths, n.acts, n.bias) for n in arch.nets]
        a = make_arch(arch.kind, nets, arch.has_b0, keep)
        d = hmc_data()
        if arch.kind == "mlp":
            d.x = _ptr(problem.x, keep, np.float32)
            d.y = _ptr(problem.y, keep, np.float32)
            d.n = int(problem.x.shape[0])
        else:
            d.u = _ptr(problem.u, keep, np.float32)
            d.q = _ptr(problem.q, keep, np.float32)
            d.v = _ptr(problem.v, keep, np.float32)
            # n_c = rows of v (all conditions; in the points_xb layout u holds this rank's block)
            d.n_c, d.n_x = int(problem.v.shape[0]), int(problem.v.shape[1])
            d.q_per_pair = int(len(problem.q.shape) == 3)  # unaligned: q [n_c, n_x, d_t]
        d.n_global = int(n_global)
        c = hmc_config()
        c.frozen = _ptr(problem.frozen, keep, np.float32)
        c.idx = _ptr(problem.idx, keep, np.int32)
        c.P = int(problem.frozen.shape[0])
        c.k = int(problem.idx.shape[0])
        c.noise_sigma = float(problem.noise_sigma)
        c.prior_sigma = float(problem.prior_sigma)
        c.inv_mass = _ptr(problem.inv_mass, keep, np.float32) if problem.inv_mass is not None else None
        c.seed = int(problem.seed)
        C = int(n_chains if n_chains is not None else problem.n_chains)
        c.n_chains = C
        ids = chain_ids if chain_ids is not None else getattr(problem, "chain_ids", None)
        if ids is not None:
            ids = np.asarray(ids, dtype=np.uint32)[:C]
            if ids.shape[0] < C:
                ids = None
        c.chain_ids = _ptr(ids, keep, np.uint32) if ids is not None else None
        c.mode = MODE[mode]
        c.rank, c.world = int(rank), int(world)
        c.shard = SHARD[shard]
        c.exchange = {"nccl": 0, "emulated": 1, "local": 2}[exchange]
        if nccl_id is not None:
            idbuf = (ctypes.c_uint8 * 128)(*nccl_id)
            keep.append(idbuf)
            c.nccl_id = ctypes.addressof(idbuf)
        self.ctx = hmc_setup(a, d, c)
        self.C, self.k, self.P = C, c.k, c.P
        _CTX_SHAPE[self.ctx] = (C, int(c.k))
        self._n_out = int(d.n) if arch.kind == "mlp" else int(d.n_c * d.n_x)

    def close(self):
        if self.ctx:
            _CTX_SHAPE.pop(self.ctx, None)
            hmc_destroy(self.ctx)
            self.ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()
