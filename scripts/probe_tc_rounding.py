"""Dev probe (not a test): rounding behaviour of tcgen05 kind::tf32 accumulation through the
engine's debug GEMM, and error growth with K for random data (tc vs SIMT vs fp64)."""
import os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2507_14652_b200 import abi

M, N, K = 128, 32, 32
def run(engine, A, B):
    M, K = A.shape; N = B.shape[1]
    tA = torch.as_tensor(np.ascontiguousarray(A, dtype=np.float32), device="cuda")
    tB = torch.as_tensor(np.ascontiguousarray(B.T, dtype=np.float32), device="cuda")
    tC = torch.zeros(M, N, device="cuda")
    abi.hmc_debug_gemm(engine, 1, 1, M, N, K, 1, tA, K, M * K, tB, K, K * N, tC, N, M * N)
    torch.cuda.synchronize()
    return tC.cpu().numpy()

d = 1.5 * 2.0 ** -24
cases = {
    "cross_group +1.5*2^-24": [(0, 1.0), (8, d)],
    "within_group +1.5*2^-24": [(0, 1.0), (1, d)],
    "small_first": [(0, d), (8, 1.0)],
    "cross_group -1.5*2^-24": [(0, 1.0), (8, -d)],
    "within_group -1.5*2^-24": [(0, 1.0), (1, -d)],
    "31 x 2^-24 spread": [(0, 1.0)] + [(k, 2.0 ** -24) for k in range(1, 32)],
    "1 + 2^-24 then 2^-24 x3 cross": [(0, 1.0), (8, 2.0 ** -24), (16, 2.0 ** -24), (24, 2.0 ** -24)],
    "1 + 0.75ulp within group 8 terms": [(0, 1.0)] + [(k, 0.75 * 2.0 ** -23 / 7) for k in range(1, 8)],
}
for name, terms in cases.items():
    A = np.zeros((M, K), np.float32); B = np.zeros((K, N), np.float32)
    exact = 0.0
    for k, v in terms:
        A[:, k] = v; B[k, :] = 1.0; exact += float(np.float32(v))
    c_tc = run(1, A, B)[0, 0]; c_s = run(0, A, B)[0, 0]
    print(f"{name:40s} exact {exact!r:24} rn32 {np.float32(exact).view(np.uint32):#x} tc {np.float32(c_tc).view(np.uint32):#x} simt {np.float32(c_s).view(np.uint32):#x}", flush=True)

g = np.random.default_rng(0)
for K in [32, 64, 256, 1024, 4096, 16384]:
    for dist in ["normal", "positive"]:
        A = g.normal(size=(128, K)) if dist == "normal" else g.uniform(0, 1, size=(128, K))
        B = g.normal(size=(K, 64)) if dist == "normal" else g.uniform(0, 1, size=(K, 64))
        A = A.astype(np.float32); B = B.astype(np.float32)
        ref = A.astype(np.float64) @ B.astype(np.float64)
        sc = np.abs(A.astype(np.float64)) @ np.abs(B.astype(np.float64))
        for eng in [0, 1]:
            C = run(eng, A, B).astype(np.float64)
            e = (C - ref) / sc
            print(f"K={K:6d} {dist:8s} {'tc  ' if eng else 'simt'} err/|A||B| rms {np.sqrt(np.mean(e**2)):.2e} max {np.abs(e).max():.2e} mean {e.mean():+.2e}", flush=True)
