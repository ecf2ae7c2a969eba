"""Dev diagnostic: CTA-0 timeline of a production tcgen05 GEMM variant inside hmc_grad on cfg5
(HMC_TC_PROF = 2 + variant id; variant 0 = forward with pre-split weights)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from hmcdata import make_problem
from paper_2507_14652_b200 import abi
prob = make_problem("cfg5")
C, k = prob.n_chains, prob.k
with abi.Context(prob) as c:
    T = torch.as_tensor(np.repeat(prob.frozen[prob.idx][None], C, 0).astype(np.float32), device="cuda")
    LP = torch.empty(C, dtype=torch.float64, device="cuda"); G = torch.empty(C, k, device="cuda")
    for _ in range(2):
        abi.hmc_grad(c.ctx, T, LP, G)
    torch.cuda.synchronize()
tl = abi.hmc_debug_tc_timeline()
t0 = tl[1, 0]
names = ["B_tma_iss", "tempty_ok", "fullop_ok", "issued", "convAll_B", "epiAll_fold", "convAll_A", "convAll_pub"]
print("variant", int(os.environ["HMC_TC_PROF"]) - 2)
print("kb  " + " ".join(f"{n:>10s}" for n in names))
for j in range(0, 24):
    print(f"{j:3d} " + " ".join(f"{(tl[i, j] - t0) if tl[i, j] else 0:10d}" for i in range(8)))
d = np.diff(tl[3, 8:120])
print("issue period median", np.median(d))
# converter warp 0, per K block: A landed -> A split -> slot free -> TMEM st issued -> B landed ->
# B split -> st done -> fence -> arrive (clocks between consecutive phases)
ph = ["A_split", "slot", "st_iss", "B_wait", "B_split", "st_done", "fence", "arrive", "->nextA"]
print("conv0 " + " ".join(f"{n:>8s}" for n in ph))
for j in range(8, 24):
    row = [tl[8, j] - tl[6, j]] + [tl[i + 1, j] - tl[i, j] for i in range(8, 15)] + [tl[6, j + 1] - tl[15, j]]
    print(f"{j:3d}   " + " ".join(f"{v:8d}" for v in row))
# epilogue warp 0, per K block: partial ready -> folded -> released -> emitted -> next ready
print("epi0    wait_tf     fold  release  emit_rg emit_out")
for j in range(8, 24):
    w = tl[16, j] - tl[19, j - 1]
    er = (tl[23, j] - tl[18, j]) if tl[23, j] else 0
    eo = (tl[19, j] - tl[23, j]) if tl[23, j] else tl[19, j] - tl[18, j]
    print(f"{j:3d}   " + " ".join(f"{v:8d}" for v in [w, tl[17, j] - tl[16, j], tl[18, j] - tl[17, j], er, eo]))
print("tile ends (kb, flush, bias/xfull, park):")
for j in range(0, 64):
    if tl[20, j]:
        print(f"{j:3d}   {tl[20, j] - tl[19, j]:8d} {tl[21, j] - tl[20, j]:8d} {tl[22, j] - tl[21, j]:8d}")
