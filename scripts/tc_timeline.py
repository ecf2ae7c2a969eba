"""Dev diagnostic: CTA-0 pipeline timeline of one tcgen05 GEMM (HMC_TC_PROF=2) via the debug GEMM:
C = A B with M=2048, N=256, K=256 (the cfg5 trunk forward shape), 64 chains."""
import os, sys
os.environ.setdefault("HMC_TC_PROF", "2")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2507_14652_b200 import abi
M, N, K, B = int(os.environ.get("TL_M", 2048)), int(os.environ.get("TL_N", 256)), int(os.environ.get("TL_K", 256)), int(os.environ.get("TL_B", 64))
akm, bkm = os.environ.get("TL_AKM", "1") == "1", os.environ.get("TL_BKM", "1") == "1"
A = torch.randn(B * M * K, device="cuda"); Bm = torch.randn(B * K * N, device="cuda"); C = torch.zeros(B * M * N, device="cuda")
lda = K if akm else M; ldb = K if bkm else N
abi.hmc_debug_tc_profile(reset=True)
for _ in range(3):
    abi.hmc_debug_gemm(1, akm, bkm, M, N, K, B, A, lda, M * K, Bm, ldb, K * N, C, N, M * N)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(); abi.hmc_debug_gemm(1, akm, bkm, M, N, K, B, A, lda, M * K, Bm, ldb, K * N, C, N, M * N); e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1)
print(f"M={M} N={N} K={K} batch={B}: {ms*1e3:.1f} us, {2*M*N*K*B/ms/1e9:.1f} TFLOP/s")
tl = abi.hmc_debug_tc_timeline()
t0 = tl[1, 0]
names = ["B_tma_iss", "tempty_ok", "fullop_ok", "issued", "convAll_B", "epiAll_fold", "convAll_A", "convAll_pub"]
print("kb  " + " ".join(f"{n:>10s}" for n in names))
for j in range(0, int(os.environ.get('TL_ROWS', 48))):
    print(f"{j:3d} " + " ".join(f"{(tl[i, j] - t0) if tl[i, j] else 0:10d}" for i in range(8)))
d = np.diff(tl[3, 8:200])
print("row0 (raw):", [int(v) for v in tl[:, 0]])
print("issue period (kb 8..200): mean", d.mean(), "median", np.median(d))
