"""Dev (make DEV=1 build): per-phase cycles of the narrow engine's CTA 0 over one trajectory."""
import ctypes, os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from hmcdata import make_problem
from paper_2507_14652_b200 import abi
cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
prob = make_problem(cfg)
L = abi.lib()
L.hmc_debug_nw_profile.argtypes = [ctypes.c_void_p, ctypes.c_int32]
out = (ctypes.c_uint64 * 10)()
with abi.Context(prob) as c:
    C, k = prob.n_chains, prob.k
    T = torch.as_tensor(np.repeat(prob.frozen[prob.idx][None], C, 0), device="cuda").contiguous()
    LP = torch.empty(C, dtype=torch.float64, device="cuda"); G = torch.empty(C, k, device="cuda")
    abi.hmc_grad(c.ctx, T, LP, G)
    abi.hmc_trajectory(c.ctx, T, LP, G, prob.eps, prob.L, 0)
    torch.cuda.synchronize()
    L.hmc_debug_nw_profile(out, 1)
    abi.hmc_trajectory(c.ctx, T, LP, G, prob.eps, prob.L, 1)
    torch.cuda.synchronize()
    L.hmc_debug_nw_profile(out, 1)
v = list(out)
names = ["forward", "output", "push", "barrier1", "reduce+update", "barrier2", "tail", "bwd:dgrad+misc", "bwd:wgrad"]
v[2], v[7] = v[2] + v[7] - v[7], v[7]  # (slot 2 = the push after the backward)
tot = sum(v[:9])
print(abi.hmc_engine_info(c.ctx) if False else cfg, "cycles per step (CTA 0):")
for n, x in zip(names, v[:9]):
    print(f"  {n:14s} {x / prob.L:10.0f}  {100 * x / max(tot, 1):5.1f}%")
