"""Dev diagnostic: where one small tcgen05 GEMM (one tile per CTA, few K blocks: the cfg4 shapes)
spends its latency.  CTA-0 timestamps of the debug GEMM (variant 7; dev build, HMC_TC_PROF = 9)
relative to kernel entry, in SM clocks."""
import os, sys
os.environ.setdefault("HMC_TC_PROF", "9")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2507_14652_b200 import abi
M, N, K, B = (int(os.environ.get(k, d)) for k, d in (("TL_M", 1000), ("TL_N", 128), ("TL_K", 128), ("TL_B", 16)))
A = torch.randn(B * M * K, device="cuda"); Bm = torch.randn(B * K * N, device="cuda"); C = torch.zeros(B * M * N, device="cuda")
def run(n=1):
    for _ in range(n):
        abi.hmc_debug_gemm(1, True, True, M, N, K, B, A, K, M * K, Bm, K, K * N, C, N, M * N)
run(3); torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(); run(1); e1.record(); torch.cuda.synchronize()
print(f"M={M} N={N} K={K} batch={B}: single launch {e0.elapsed_time(e1)*1e3:.1f} us")
e0.record(); run(20); e1.record(); torch.cuda.synchronize()
print(f"20 back-to-back launches (PDL): {e0.elapsed_time(e1)*1e3/20:.1f} us each")
tl = abi.hmc_debug_tc_timeline().astype(np.int64)
n = tl.shape[1]
t_in = tl[0, n - 1]
print("kernel entry 0, prologue end", tl[0, n - 2] - t_in, ", warp-0 body end", tl[0, n - 3] - t_in, ", CTA exit", tl[0, n - 4] - t_in)
names = ["B_tma_iss", "tempty_ok", "fullop_ok", "mma_issued", "convAll_B", "epiAll_fold", "convAll_A", "convAll_pub",
         "c0_Asplit", "c0_slot", "c0_st_iss", "c0_Bwait", "c0_Bsplit", "c0_st_done", "c0_fence", "c0_arrive",
         "e0_tfull", "e0_folded", "e0_release", "e0_emitted", "tile_flush", "tile_bias", "tile_park", "emit_regs"]
nk = (K + 31) // 32
for i, nm in enumerate(names):
    print(f"{i:2d} {nm:12s} " + " ".join(f"{(tl[i, j] - t_in) if tl[i, j] else 0:8d}" for j in range(min(nk, 8))))
