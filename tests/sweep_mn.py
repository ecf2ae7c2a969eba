"""Device check of MN-major tcgen05 descriptor encodings (dev tool, not a test)."""
import itertools, os, subprocess, sys, json
combos = []
for tma, lay, sbo, kstep in itertools.product([32, 128], [1, 2], [512, 1024], [1024, 512]):
    combos.append(dict(HMC_MN_TMA=str(tma), HMC_MN_LAYOUT=str(lay), HMC_MN_SBO=str(sbo), HMC_MN_KSTEP=str(kstep)))
code = r'''
import numpy as np, torch, sys
sys.path.insert(0, ".")
from paper_2507_14652_b200 import abi
res = {}
for akm, bkm, M, N, K in [(True, False, 256, 256, 64), (False, True, 256, 128, 64), (False, False, 128, 128, 32)]:
    g = np.random.default_rng(0)
    A = g.normal(size=(M, K)).astype(np.float32); B = g.normal(size=(K, N)).astype(np.float32)
    Ad, lda = (A, K) if akm else (np.ascontiguousarray(A.T), M)
    Bd, ldb = (np.ascontiguousarray(B.T), K) if bkm else (B, N)
    tA = torch.as_tensor(Ad, device="cuda").contiguous(); tB = torch.as_tensor(Bd, device="cuda").contiguous()
    tC = torch.zeros(M, N, device="cuda")
    abi.hmc_debug_gemm(1, akm, bkm, M, N, K, 1, tA, lda, M*K, tB, ldb, K*N, tC, N, M*N)
    torch.cuda.synchronize()
    ref = A.astype(np.float64) @ B.astype(np.float64)
    res[f"{int(akm)}{int(bkm)}"] = float(np.abs(tC.cpu().numpy() - ref).max() / np.abs(ref).max())
print("RES", res)
'''
for c in combos:
    env = dict(os.environ, **c)
    try:
        out = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=60)
        line = [l for l in out.stdout.splitlines() if l.startswith("RES")]
        print(json.dumps(c), line[0] if line else ("FAIL " + out.stderr[-300:]), flush=True)
    except subprocess.TimeoutExpired:
        print(json.dumps(c), "TIMEOUT", flush=True)
